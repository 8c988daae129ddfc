#!/usr/bin/env python
"""Benchmark: fwd+inv SGL transforms/s at B=128, fp64 (BASELINE.json metric).

One step = one inverse transform (ifsglft) of a coefficient vector followed by one
forward transform (fsglft) of the resulting grid -- the reference's timed round
trip (tools/commands.cpp:152-177) -- for `--batch` functions.
Default workload: BASELINE config C3, B = 128, one complex function per step,
f_nlm iid complex normal (synthetic, numpy PCG64 seed 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  `value` is device-timed (inputs resident in HBM,
CUDA events on the launch stream, max over ranks); `e2e` is the same round trip
through the public host API (numpy in pinned host memory, H2D/D2H inside the
timed region).  `--impl reference` times the reference's own CPU implementation
(oracle/_ref, compiled from /root/reference; else the oracle port) on the host.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

FP64_PEAK_TFLOPS = 37.1  # measured DMMA m8n8k4 peak on this pool's B200 (profiles/fp64_peak_r01.txt)


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def config_id(B, nb):
    """BASELINE.json config label for a (B, functions per step) workload."""
    return {(16, 1): "C1", (64, 64): "C2", (128, 1): "C3", (256, 1): "C4"}.get((B, nb), "custom")


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def complex_normal(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2.0)


def real_valued_coeffs(rng, B, shape):
    """BASELINE config C5: m > 0 complex normal x exp(-n/8), m = 0 real normal x
    exp(-n/8), f_{n,l,-m} = (-1)^m conj(f_nlm)."""
    n_of, l_of, m_of = [], [], []
    for n in range(1, B + 1):
        for l in range(n):
            for m in range(-l, l + 1):
                n_of.append(n)
                l_of.append(l)
                m_of.append(m)
    n_of, l_of, m_of = (np.array(a) for a in (n_of, l_of, m_of))
    c = complex_normal(rng, shape + (len(n_of),)) * np.exp(-n_of / 8.0)
    zero = m_of == 0
    c[..., zero] = c[..., zero].real * np.sqrt(2.0)
    neg = np.nonzero(m_of < 0)[0]
    mirror = neg - 2 * m_of[neg]  # omega(n, l, -m) = omega(n, l, m) - 2m
    c[..., neg] = ((-1.0) ** m_of[neg]) * np.conj(c[..., mirror])
    return c


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while the timed region runs."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device_index: int):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._ok:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ reference arm
def reference_arm(args, rank, world):
    if rank != 0:
        return
    from oracle_bindings import Oracle, Reference, coefficient_count

    B = args.B
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(0)
    c = complex_normal(rng, coefficient_count(B))
    kind = "reference"
    try:
        impl = Reference(B)
        note = "reference fsglft/ifsglft (oracle/_ref, built from /root/reference) threads=0"
        if B >= 128:
            note += "; NOTE: reference output is numerically invalid at B>=128 (M_lm underflow), timing only"
    except Exception as e:  # reference not built here
        impl = Oracle(B)
        kind = "port"
        note = f"oracle port (C restatement, OpenMP) -- reference unavailable: {e}"
    # one untimed warm-up round trip (plan caches, page faults); the reference's
    # CPU round trip at B=128 takes ~1 s, so the timed steps are capped at ~120 s
    t0 = time.perf_counter()
    impl.forward(impl.inverse(c, threads=0), threads=0)
    est = time.perf_counter() - t0
    run = max(1, min(args.steps, int(120.0 / max(est, 1e-6))))
    t_all = time.perf_counter()
    for _ in range(run):
        g = impl.inverse(c, threads=0)
        impl.forward(g, threads=0)
    total = time.perf_counter() - t_all
    ms = 1000.0 * total / run
    note += f"; timed {run} of the requested {args.steps} steps (each step = one fwd+inv round trip)"
    value = args.batch / (ms / 1000.0) if args.batch == 1 else 1.0 / (ms / 1000.0)
    line = {
        "impl": "reference", "metric": f"fwd+inv SGL transforms/s at B={B} fp64", "value": value,
        "unit": "transforms/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: iid complex normal coefficients (numpy PCG64 seed 0)",
        "config": {"workload": f"C3: B={B}, 1 function, ifsglft then fsglft", "B": B, "batch": 1},
        "cpu_baseline": {"value": value, "unit": "transforms/s", "cores": cores, "kind": kind,
                         "sample": f"{args.steps} round trips, {note}"},
        "e2e": {"value": value, "unit": "transforms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(B, budget_s=12.0):
    """Reference (or oracle port) round trips on the host cores, bounded to ~budget_s."""
    from oracle_bindings import Oracle, Reference, coefficient_count

    rng = np.random.default_rng(0)
    c = complex_normal(rng, coefficient_count(B))
    kind = "reference"
    try:
        impl = Reference(B)
        note = "reference fsglft/ifsglft, threads=0 (all cores)"
        if B >= 128:
            note += "; reference output invalid at B>=128 (M_lm underflow) -- timing only"
    except Exception:
        impl = Oracle(B)
        kind = "port"
        note = "oracle C restatement, OpenMP all cores"
    impl.forward(impl.inverse(c, threads=0), threads=0)  # warm
    n = 0
    t0 = time.perf_counter()
    while True:
        impl.forward(impl.inverse(c, threads=0), threads=0)
        n += 1
        if time.perf_counter() - t0 > budget_s or n >= 200:
            break
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "transforms/s", "cores": os.cpu_count() or 1, "kind": kind,
            "sample": f"{n} fwd+inv round trips at B={B} in {dt:.1f} s; {note}"}


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--B", type=int, default=128)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="split", choices=["split", "replicas"],
                    help="N>1: split one transform by shells / (l, m) (strong scaling, default) "
                         "or run independent replicas (weak scaling)")
    ap.add_argument("--force-split", action="store_true", help="run the split path even at N=1 (testing)")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="split mode: stage exchange fused into the kernels (NVLink peer stores) or NCCL all-to-all")
    ap.add_argument("--real", action="store_true",
                    help="real-valued functions through the real fast path (config C5: f_{nl,-m} = (-1)^m conj f_nlm, "
                         "|f_nlm| ~ exp(-n/8))")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local = env_rank()

    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if (world > 1 and args.mode == "split") or args.force_split:
        split_arm(args, rank, world, local)
        return

    import torch

    import paper_1604_05140_b200 as sgl
    from paper_1604_05140_b200 import workload as wl

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    B, nb = args.B, args.batch
    Om, Ps = sgl.coefficient_count(B), sgl.sample_count(B)
    plan = sgl.TransformPlan.compute(B, device=local)
    L = sgl.lib()
    L.sglgpu_profile_begin.argtypes = [ctypes.c_void_p]
    L.sglgpu_profile_end.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]

    # inputs resident in HBM; rotate over enough distinct coefficient buffers that
    # each step's input is not L2 resident (>= 2 x 126 MB of inputs)
    l2 = 126e6
    nrot = max(2, min(64, math.ceil(2 * l2 / (16 * Om * nb))))
    rng = np.random.default_rng(rank)
    if args.real:
        nrot = max(2, min(nrot, 8))
        cin = torch.from_numpy(real_valued_coeffs(rng, B, (nrot, nb))).cuda()
    else:
        cin = torch.from_numpy(complex_normal(rng, (nrot, nb, Om))).cuda()
    grid = torch.empty((nb, Ps), dtype=torch.float64 if args.real else torch.complex128, device="cuda")
    cout = torch.empty((nb, Om), dtype=torch.complex128, device="cuda")
    # a dedicated (non-default) stream: the library replays CUDA graphs of
    # transforms up to 2 x 128^3 samples on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    # The headline pass runs without per-stage events (an event record between
    # kernels costs ~5 us of GPU time each, ~30 us per B = 128 round trip, and
    # disables graph replay); the stage times and the roofline come from a second
    # timed pass over the same steps with CUDA events around every stage launch.
    graphs = (B ** 3) * nb <= 2 * 128 ** 3
    live_profile = False

    inv = sgl.ifsglft_real_batch if args.real else sgl.ifsglft_batch
    fwd = sgl.fsglft_real_batch if args.real else sgl.fsglft_batch

    def step(s):
        inv(plan, cin[s % nrot], out=grid)
        fwd(plan, grid, out=cout)

    for s in range(max(args.warmup, 2 * nrot + 2 if graphs else 0)):  # graph capture starts at the second call per input: every input twice
        step(s)
    torch.cuda.synchronize()
    # correctness guard on the warm-up output
    wl_last = max(args.warmup, 2 * nrot + 2 if graphs else 0) - 1
    err = float((cout - cin[wl_last % nrot]).abs().max() / cin[wl_last % nrot].abs().max())

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stage_ms = np.zeros(6)
    stage_n = np.zeros(6, dtype=np.int32)
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        if live_profile:
            assert L.sglgpu_profile_begin(plan.handle) == 0
        ev0.record(stream)
        for s in range(args.steps):
            step(s)
        ev1.record(stream)
        torch.cuda.synchronize()
        if live_profile:
            assert L.sglgpu_profile_end(plan.handle, stage_ms.ctypes.data, stage_n.ctypes.data) == 0
        if dist:
            dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if not live_profile:
        torch.cuda.synchronize()
        assert L.sglgpu_profile_begin(plan.handle) == 0
        for s in range(args.steps):
            step(s)
        torch.cuda.synchronize()
        assert L.sglgpu_profile_end(plan.handle, stage_ms.ctypes.data, stage_n.ctypes.data) == 0
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * nb / (ms / 1000.0)
    gpu_launches = int(stage_n.sum())

    # ---- e2e through the public host API (pinned host buffers, copies timed)
    hc = torch.empty((nb, Om), dtype=torch.complex128).pin_memory().numpy()
    hc[:] = cin[0].cpu().numpy()
    hg = torch.empty((nb, Ps), dtype=torch.float64 if args.real else torch.complex128).pin_memory().numpy()
    hb = torch.empty((nb, Om), dtype=torch.complex128).pin_memory().numpy()
    inv(plan, hc, out=hg)
    fwd(plan, hg, out=hb)
    ke = args.e2e_steps
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(ke):
        inv(plan, hc, out=hg)
        fwd(plan, hg, out=hb)
    e2e_ms = 1000.0 * (time.perf_counter() - t0) / ke
    if dist:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_err = float(np.abs(hb - hc).max() / np.abs(hc).max())

    # ---- roofline of the dominant kernel (live CUDA-event times from the timed region)
    peaks = load_peaks()
    work = wl.stage_work(B)
    dom = int(np.argmax(stage_ms))
    per_launch_ms = stage_ms[dom] / max(1, stage_n[dom])
    flops, nbytes = work[dom]
    # algorithmic work of one launch = per-step work / launches per step
    lps = max(1, int(stage_n[dom]) // args.steps)
    flops *= nb / lps
    nbytes *= nb / lps
    stage_info = {}
    for s in range(6):
        if stage_n[s]:
            t_ms = stage_ms[s] / args.steps  # per step (a stage may be split into several launches)
            tf = work[s][0] * nb / (t_ms * 1e-3) / 1e12
            gb = work[s][1] * nb / (t_ms * 1e-3) / 1e9
            hbm = s in (0, 5)  # the azimuthal kernels are HBM-bound, the contractions FP64-bound
            stage_info[wl.STAGE_NAMES[s]] = {
                "ms": round(t_ms, 5), "launches_per_step": int(stage_n[s]) // args.steps,
                "tflops": round(tf, 3), "gbs": round(gb, 1),
                "bound": "hbm" if hbm else "tensor",
                "roofline_frac": round(gb / peaks["hbm_gbs"] if hbm else tf / FP64_PEAK_TFLOPS, 3),
                "share": round(stage_ms[s] / stage_ms.sum(), 4),
            }
    if dom in (0, 5):
        achieved = nbytes / (per_launch_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                "kernel": wl.STAGE_NAMES[dom], "algorithmic_bytes_per_launch": nbytes,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)"}
    else:
        achieved = flops / (per_launch_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None,
                "kernel": wl.STAGE_NAMES[dom], "algorithmic_flops_per_launch": flops,
                "peak_source": "measured fp64 DMMA (mma.sync m8n8k4) peak, profiles/fp64_peak_r01.txt; "
                               "MEASURED_PEAKS.json has no fp64 entry"}
    roof["launch_ms"] = per_launch_ms
    # DRAM traffic of this kernel from the committed ncu --set full capture (B = 128)
    try:
        with open(os.path.join(REPO, "profiles", "r01_traffic.json")) as f:
            tr = json.load(f)["bytes"]
        knames = {0: [f"void az_forward_kernel<{2 * B}>"], 1: ["void gemm_dmma_kernel<LegFwdTma>", "void gemm_dmma_kernel<LegFwd>"],
                  2: ["void gemm_dmma_kernel<RadFwd>"], 3: ["void gemm_dmma_kernel<RadInv>"],
                  4: ["void gemm_dmma_kernel<LegInvSeq>", "void gemm_dmma_kernel<LegInv>"],
                  5: [f"void az_inverse_kernel<{2 * B}>"]}[dom]
        kname = next((k for k in knames if k in tr), None)
        if B == 128 and nb == 1 and kname is not None:
            roof["traffic"] = tr[kname]
            roof["traffic_source"] = "profiles/r01_ncu_full.txt (dram__bytes_read.sum + dram__bytes_write.sum)"
    except (OSError, KeyError, ValueError):
        pass
    roof["timing"] = ("live: CUDA events around each stage launch inside the timed region" if live_profile else
                      "live: CUDA events around each stage launch (eager launches) in a second timed pass of "
                      "the same steps, right after the headline pass")
    whole = 2 * wl.f_fwd(B) * nb / (ms * 1e-3) / 1e12

    line = {
        "metric": f"fwd+inv SGL transforms/s at B={B} fp64", "value": value, "unit": "transforms/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: iid complex normal coefficients (numpy PCG64, seed = rank)",
        "config": {"workload": (f"C5: B={B}, {nb} real-valued functions per step per GPU (real fast path)"
                                if args.real else f"{config_id(B, nb)}: B={B}, {nb} function(s) per step per GPU, "
                                                  "ifsglft then fsglft"),
                   "B": B, "batch_per_gpu": nb, "parallelism": f"replicas x{world}" if world > 1 else "single",
                   "l2": f"inputs rotated over {nrot} coefficient buffers ({nrot * 16 * Om * nb / 1e6:.0f} MB) "
                         f"and every step writes/reads a {16 * Ps * nb / 2**20:.0f} MiB grid (> 126 MB L2)"},
        "e2e": {"value": world * nb / (e2e_ms / 1000.0), "unit": "transforms/s",
                "h2d_bytes_per_step": (16 * Om + (8 if args.real else 16) * Ps) * nb,
                "d2h_bytes_per_step": ((8 if args.real else 16) * Ps + 16 * Om) * nb,
                "ms_per_step": e2e_ms, "api": "paper_1604_05140_b200.ifsglft_batch/fsglft_batch (C ABI, host mem)"},
        "gpu_launches": gpu_launches,
        "roofline": roof,
        "transform_fp64_tflops": whole,
        "transform_roofline_frac": whole / FP64_PEAK_TFLOPS,
        "stages": stage_info,
        "clocks": clk.summary(),
        "roundtrip_normwise_err": max(err, e2e_err),
    }
    if not (line["roundtrip_normwise_err"] < 1e-10):
        raise SystemExit(f"bench: round trip failed (normwise error {line['roundtrip_normwise_err']:.3e}); "
                         "refusing to report a timing of wrong results")
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(B)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def split_arm(args, rank, world, local):
    """N > 1: one B = 128 transform per step split over the ranks -- spherical stage
    by radial shell, radial stage by degree range, NCCL all-to-all in between
    (paper_1604_05140_b200.distributed).  Strong scaling."""
    import torch
    import torch.distributed as dist

    import paper_1604_05140_b200 as sgl
    from paper_1604_05140_b200 import workload as wl
    from paper_1604_05140_b200.distributed import (CudaStages, Partition, PeerBuffers, fsglft_distributed,
                                                   fsglft_distributed_fused, ifsglft_distributed,
                                                   ifsglft_distributed_fused)

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B, nb = args.B, args.batch
    Om, Ps = sgl.coefficient_count(B), sgl.sample_count(B)
    plan = sgl.TransformPlan.compute(B, device=local)
    st = CudaStages(plan)
    part = Partition.make(B, world)
    nrot = max(2, min(64, math.ceil(2 * 126e6 / (16 * Om * nb))))
    rng = np.random.default_rng(0)  # same coefficients on every rank
    cin = torch.from_numpy(complex_normal(rng, (nrot, nb, Om))).cuda()
    stream = torch.cuda.current_stream()

    # the exchange: fused into the stage epilogues (peer stores into CUDA-IPC-mapped
    # receive buffers) unless --exchange nccl or the peers cannot be mapped
    exchange, why = args.exchange, ""
    peers = None
    if exchange == "fused":
        try:
            peers = PeerBuffers.exchange(part, nb, dist)
        except Exception as e:  # noqa: BLE001 -- e.g. IPC not permitted: fall back to the NCCL all-to-all
            exchange, why = "nccl", f"fused exchange unavailable: {e}"
        flag = torch.tensor([0.0 if exchange == "fused" else 1.0], device="cuda")
        dist.all_reduce(flag)  # every rank must take the same path
        if flag.item() > 0 and exchange == "fused":
            exchange, why = "nccl", "fused exchange unavailable on a peer"
    inv_d = (lambda c: ifsglft_distributed_fused(c, part, st, peers, dist, batch=nb)) if exchange == "fused" else \
        (lambda c: ifsglft_distributed(c, part, st, dist, batch=nb))
    fwd_d = (lambda x: fsglft_distributed_fused(x, part, st, peers, dist, batch=nb)) if exchange == "fused" else \
        (lambda x: fsglft_distributed(x, part, st, dist, batch=nb))

    def step(s):
        return fwd_d(inv_d(cin[s % nrot]).view(nb, -1))

    for s in range(args.warmup):
        out = step(s)
    torch.cuda.synchronize()
    ref = cin[(args.warmup - 1) % nrot]
    err = float((out - ref).abs().max() / ref.abs().max())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for s in range(args.steps):
            step(s)
        ev1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = nb / (ms / 1000.0)
    # e2e: host coefficients in, host shell slice out and back in, host coefficients out
    sc = part.shells_per_rank
    hc = torch.empty((nb, Om), dtype=torch.complex128).pin_memory()
    hc.copy_(cin[0].cpu())
    hloc = torch.empty((nb, sc * 4 * B * B), dtype=torch.complex128).pin_memory()
    hout = torch.empty((nb, Om), dtype=torch.complex128).pin_memory()
    ke = args.e2e_steps
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(ke):
        loc = inv_d(hc.cuda(non_blocking=True))
        hloc.copy_(loc.view(nb, -1), non_blocking=True)
        c2 = fwd_d(hloc.cuda(non_blocking=True))
        hout.copy_(c2, non_blocking=True)
        torch.cuda.synchronize()
    e2e_ms = 1000.0 * (time.perf_counter() - t0) / ke
    t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    whole = 2 * wl.f_fwd(B) * nb / (ms * 1e-3) / 1e12
    line = {
        "metric": f"fwd+inv SGL transforms/s at B={B} fp64", "value": value, "unit": "transforms/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: iid complex normal coefficients (numpy PCG64, seed 0)",
        "config": {"workload": f"C3: B={B}, {nb} function(s) per step split over {world} GPUs "
                               "(shells / degree ranges, " + ("exchange fused into the stage epilogues: NVLink "
                               "peer stores" if exchange == "fused" else "NCCL all-to-all") + ")",
                   "exchange": exchange + (f" ({why})" if why else ""),
                   "B": B, "batch": nb, "parallelism": f"shell/(l,m) split x{world}",
                   "l2": f"inputs rotated over {nrot} buffers; per-step grid {16 * Ps * nb / 2**20:.0f} MiB > L2"},
        "e2e": {"value": nb / (e2e_ms / 1000.0), "unit": "transforms/s",
                "h2d_bytes_per_step": 16 * (Om + sc * 4 * B * B) * nb,
                "d2h_bytes_per_step": 16 * (sc * 4 * B * B + Om) * nb, "ms_per_step": e2e_ms,
                "api": "paper_1604_05140_b200.distributed.{ifsglft,fsglft}_distributed" +
                       ("_fused" if exchange == "fused" else "")},
        "gpu_launches": 6 * args.steps,
        "transform_fp64_tflops": whole,
        "transform_roofline_frac": whole / FP64_PEAK_TFLOPS,
        "clocks": clk.summary(),
        "roundtrip_normwise_err": err,
    }
    if not (err < 1e-10):
        raise SystemExit(f"bench: distributed round trip failed (normwise error {err:.3e})")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if peers is not None:
        torch.cuda.synchronize()
        dist.barrier()
        peers.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
