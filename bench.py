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
TRAFFIC_FILE = "r02g_traffic.json"  # per-kernel DRAM bytes of the committed ncu capture (B = 128, one function)


def KERNEL_NAMES(B):  # noqa: N802 -- ncu names of each stage's kernels
    return {0: [f"void az_forward_kernel<{2 * B}>"],
            1: ["void gemm_dmma_kernel<LegFwdTma>", "void gemm_dmma_kernel<LegFwd>"],
            2: ["void gemm_dmma_kernel<RadFwd>"], 3: ["void gemm_dmma_kernel<RadInv>"],
            4: ["void leginv_wp_kernel<64, 0>", "void leginv_wp_kernel<32, 0>", "void leginv_wp_kernel<128, 0>",
                "void leginv_wp_kernel<64>", "void gemm_dmma_kernel<LegInvSeq>", "void gemm_dmma_kernel<LegInv>"],
            5: [f"void az_inverse_kernel<{2 * B}>"],
            6: [f"void sph_fwd_fused_kernel<{2 * B}>"], 7: [f"void sph_inv_fused_kernel<{2 * B}>"]}


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def config_id(B, nb, real=False):
    """BASELINE.json config label for a (B, functions per step, real-valued) workload."""
    if real:
        return {(32, 4096): "C5"}.get((B, nb), "custom")
    return {(16, 1): "C1", (64, 64): "C2", (128, 1): "C3", (256, 1): "C4"}.get((B, nb), "custom")


def workload_config(B, nb, real):
    """The `config` dict -- identical in both arms (ours and --impl reference), so the
    driver can match the lines; run details go to the line's `setup` key."""
    kind = "real-valued" if real else "complex"
    return {"workload": f"{config_id(B, nb, real)}: B={B}, {nb} {kind} function(s) per step, ifsglft then fsglft",
            "B": B, "batch": nb, "real": bool(real)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


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


def nl_of_omega(B):
    n_of, l_of = [], []
    for n in range(1, B + 1):
        for l in range(n):
            n_of += [n] * (2 * l + 1)
            l_of += [l] * (2 * l + 1)
    return np.array(n_of), np.array(l_of)


def config_coefficients(rng, B, shape, real=False):
    """Coefficients with BASELINE.json's value distribution for the config:
    C2 (B = 64): complex normal x exp(-n/16); C4 (B = 256): complex normal x
    (1 + l)^-1; C5 (real): see real_valued_coeffs; otherwise iid complex normal."""
    if real:
        return real_valued_coeffs(rng, B, shape)
    n_of, l_of = nl_of_omega(B)
    c = complex_normal(rng, shape + (len(n_of),))
    if B == 64:
        c *= np.exp(-n_of / 16.0)
    elif B == 256:
        c /= 1.0 + l_of
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
def _input_coefficients(B, nb, real, seed=0):
    return config_coefficients(np.random.default_rng(seed), B, (nb,), real)


def cpu_reference(B, nb, real, budget_s, max_steps=None):
    """The reference's own CPU implementation of the timed round trip
    (ifsglft then fsglft, tools/commands.cpp:152-177) on this host, as BASELINE.md
    section 3 prescribes: oracle/_ref (the reference compiled from its sources)
    with threads=0 for single functions, an outer pool of nproc threads with
    threads=1 per function for batches (ref_roundtrip_batch); the oracle port
    (C restatement) only if the reference was not built.  At B >= 128 the
    reference's output is invalid (M_lm underflow), so the robust port is timed
    beside it.  Bounded to ~budget_s of CPU time: a step is one round trip of
    one function (single) or of a sample of the batch (pool)."""
    from oracle_bindings import Oracle, Reference

    cores = os.cpu_count() or 1
    kind = "reference"
    try:
        impl = Reference(B)
    except Exception as e:  # noqa: BLE001 -- reference not built on this host
        impl, kind = Oracle(B), "port"
        why = f"{e}"
    out = {"unit": "transforms/s", "cores": cores, "kind": kind, "cpu_model": cpu_model()}

    def one(obj, c, threads=0):
        obj.forward(obj.inverse(c, threads=threads), threads=threads)

    if nb == 1:
        # threads=0 (all cores) as BASELINE.md prescribes -- unless one thread is
        # faster (small B: the reference spawns threads per call, parallel.cpp:14-41)
        c = _input_coefficients(B, 1, real)[0]
        est = {}
        for th in ((0, 1) if B <= 32 else (0,)):
            one(impl, c, th)  # warm (plan caches, page faults)
            t0 = time.perf_counter()
            one(impl, c, th)
            est[th] = time.perf_counter() - t0
        th = min(est, key=est.get)
        steps = max(1, int(budget_s / max(est[th], 1e-6)))
        if max_steps:
            steps = min(steps, max_steps)
        t0 = time.perf_counter()
        for _ in range(steps):
            one(impl, c, th)
        dt = time.perf_counter() - t0
        out["value"] = steps / dt
        out["cores"] = cores if th == 0 else 1
        out["sample"] = (f"{steps} round trips of one B={B} function, fsglft/ifsglft threads={th} "
                         f"({'reference oracle/_ref' if kind == 'reference' else 'oracle port: ' + why})")
    else:
        # outer pool: sample enough functions for ~budget_s
        pool = cores
        c1 = _input_coefficients(B, pool, real)
        if kind == "reference":
            t0 = time.perf_counter()
            impl.roundtrip_batch(c1, pool)
            est = (time.perf_counter() - t0) / pool  # per function, with the pool busy
            n = int(min(nb, max(pool, budget_s / max(est, 1e-9)))) // pool * pool or pool
            c = _input_coefficients(B, n, real)
            t0 = time.perf_counter()
            impl.roundtrip_batch(c, pool)
            dt = time.perf_counter() - t0
            out["sample"] = (f"{n} of the {nb} B={B} functions of one step through an outer pool of {pool} threads, "
                             "threads=1 per function (reference oracle/_ref, ref_roundtrip_batch)")
        else:
            c = c1
            t0 = time.perf_counter()
            for f in range(pool):
                one(impl, c[f])
            dt = time.perf_counter() - t0
            n = pool
            out["sample"] = f"{n} B={B} functions, oracle port with OpenMP threads ({why})"
        out["value"] = n / dt
    if B >= 128 and kind == "reference":
        out["reference_output_valid"] = False
        out["note"] = ("reference output is numerically invalid at B >= 128 (M_lm underflow, "
                       "special_functions.cpp:81-88): timing only; port_value = the robust C restatement")
        orc = Oracle(B)
        c = _input_coefficients(B, 1, real)[0]
        one(orc, c)
        t0 = time.perf_counter()
        one(orc, c)
        out["port_value"] = 1.0 / (time.perf_counter() - t0)
    return out


def reference_arm(args, rank, world):
    """--impl reference: rank 0 times the reference's CPU implementation on the
    same workload (config dict identical to our arm's); other ranks exit."""
    if rank != 0:
        return
    B, nb = args.B, args.batch
    t_all = time.perf_counter()
    budget = max(20.0, min(150.0, 0.75 * args.steps))  # a few minutes at most for the whole run
    cb = cpu_reference(B, nb, args.real, budget, max_steps=args.steps)
    value = cb["value"]
    line = {
        "impl": "reference", "metric": f"fwd+inv SGL transforms/s at B={B} fp64", "value": value,
        "unit": "transforms/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * nb / value, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic: BASELINE.json config coefficients (numpy PCG64 seed 0)",
        "config": workload_config(B, nb, args.real),
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "transforms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup": {"wall_s": round(time.perf_counter() - t_all, 1),
                  "ms_per_step": "per step of `batch` functions, extrapolated from the timed sample"},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--B", type=int, default=128)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=32)
    ap.add_argument("--e2e-callers", type=int, default=4,
                    help="host threads issuing the e2e round trips concurrently (PCIe full duplex)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="auto", choices=["auto", "split", "replicas"],
                    help="N>1: split one transform by shells / (l, m) (strong scaling; BASELINE configs C3/C4) "
                         "or shard the batch as independent replicas (weak scaling; C2/C5); auto: split for one "
                         "function per step, replicas for batches")
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
    if args.mode == "auto":
        args.mode = "split" if args.batch == 1 and not args.real else "replicas"
    if world > 1:
        # keep NCCL's communicator log on (rank count, transport: NVLink / NVLS) for the driver
        os.environ.setdefault("NCCL_DEBUG", "INFO")
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
    cin = torch.from_numpy(config_coefficients(rng, B, (nrot, nb), args.real)).cuda()
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
    stage_ms = np.zeros(8)
    stage_n = np.zeros(8, dtype=np.int32)
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

    # ---- e2e through the public host API (pinned host buffers, copies timed).
    # Every step uploads its coefficients and its grid and downloads its grid and
    # its coefficients (the round trip through host memory).  Steps are issued by
    # `--e2e-callers` host threads calling the same plan concurrently (the library
    # runs host calls of different threads on separate streams), so one caller's
    # downloads overlap another's uploads on the full-duplex PCIe link; each
    # caller's steps are strictly sequential.  Odd-numbered callers run their
    # round trip forward-first (fsglft of their grid, then ifsglft of the
    # result), so that while an even caller downloads its grid an odd one uploads
    # its grid (measured on the box: 55.5 GB/s H2D, 57.2 D2H, 99.4 both at once;
    # callers in the same order lock into the same phase and share one
    # direction).  The single-caller figure is reported beside it.
    def make_host():
        hc = torch.empty((nb, Om), dtype=torch.complex128).pin_memory().numpy()
        hc[:] = cin[0].cpu().numpy()
        hg = torch.empty((nb, Ps), dtype=torch.float64 if args.real else torch.complex128).pin_memory().numpy()
        hb = torch.empty((nb, Om), dtype=torch.complex128).pin_memory().numpy()
        return hc, hg, hb

    def e2e_run(callers, steps_each):
        bufs = [make_host() for _ in range(callers)]
        errs = []
        # every caller warms up from its own thread (so each host slot of the
        # library -- streams, workspaces, device staging -- exists before the timed
        # region), then all start together
        start = threading.Barrier(callers + 1)
        done = threading.Barrier(callers + 1)

        def worker(i, b):
            hc, hg, hb = b
            inv(plan, hc, out=hg)
            fwd(plan, hg, out=hb)
            start.wait()
            for _ in range(steps_each):
                if i % 2 == 0:
                    inv(plan, hc, out=hg)
                    fwd(plan, hg, out=hb)
                else:
                    fwd(plan, hg, out=hb)
                    inv(plan, hb, out=hg)
            done.wait()
            errs.append(float(np.abs(hb - hc).max() / np.abs(hc).max()))

        ts = [threading.Thread(target=worker, args=(i, b)) for i, b in enumerate(bufs)]
        for t in ts:
            t.start()
        if dist:
            dist.barrier()
        start.wait()
        t0 = time.perf_counter()
        done.wait()
        ms = 1000.0 * (time.perf_counter() - t0) / (callers * steps_each)
        for t in ts:
            t.join()
        if dist:
            t = torch.tensor([ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, max(errs)

    ke = args.e2e_steps
    e2e_single_ms, e2e_err1 = e2e_run(1, ke)
    # callers share the host's pinned memory: at most ~16 GB of caller buffers
    per_caller = (16 * Om * 2 + (8 if args.real else 16) * Ps) * nb
    callers = max(1, min(args.e2e_callers, int((16 << 30) // max(1, per_caller))))
    e2e_ms, e2e_err = e2e_run(callers, max(1, (ke + callers - 1) // callers)) if callers > 1 else (e2e_single_ms, e2e_err1)
    e2e_err = max(e2e_err, e2e_err1)

    # ---- roofline of the dominant kernel (live CUDA-event times from the timed region)
    # Algorithmic work is the reference algorithm's (workload.py);
    # the real fast path does half of it (only m >= 0), so it is credited half.
    peaks = load_peaks()
    work = wl.stage_work(B)
    rscale = 0.5 if args.real else 1.0
    dom = int(np.argmax(stage_ms))
    per_launch_ms = stage_ms[dom] / max(1, stage_n[dom])
    flops, nbytes, gbytes = work[dom]
    # algorithmic work of one launch = per-step work / launches per step
    lps = max(1, int(stage_n[dom]) // args.steps)
    flops *= rscale * nb / lps
    nbytes *= rscale * nb / lps
    stage_info = {}
    for s in range(8):
        if stage_n[s]:
            t_ms = stage_ms[s] / args.steps  # per step (a stage may be split into several launches)
            tf = rscale * work[s][0] * nb / (t_ms * 1e-3) / 1e12
            gb = rscale * work[s][1] * nb / (t_ms * 1e-3) / 1e9
            gi = rscale * (work[s][1] + work[s][2]) * nb / (t_ms * 1e-3) / 1e9
            hbm = s in (0, 5)  # the azimuthal kernels are HBM-bound, the contractions (and fused stages) FP64-bound
            stage_info[wl.STAGE_NAMES[s]] = {
                "ms": round(t_ms, 5), "launches_per_step": int(stage_n[s]) // args.steps,
                "tflops": round(tf, 3), "gbs_compulsory": round(gb, 1), "gbs_with_intermediate": round(gi, 1),
                "bound": "hbm" if hbm else "fp64",
                "roofline_frac": round(gb / peaks["hbm_gbs"] if hbm else tf / FP64_PEAK_TFLOPS, 3),
                "share": round(stage_ms[s] / stage_ms.sum(), 4),
            }
    if dom in (0, 5):
        achieved = nbytes / (per_launch_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                "kernel": wl.STAGE_NAMES[dom], "algorithmic_bytes_per_launch": nbytes,
                "intermediate_bytes_per_launch": rscale * gbytes * nb / lps,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)"}
    else:
        achieved = flops / (per_launch_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None,
                "kernel": wl.STAGE_NAMES[dom], "algorithmic_flops_per_launch": flops,
                "peak_source": "builder-measured fp64 DMMA (mma.sync m8n8k4) peak, profiles/fp64_peak_r01.txt; "
                               "MEASURED_PEAKS.json has no fp64 entry"}
    roof["launch_ms"] = per_launch_ms
    # DRAM traffic of this kernel from the committed ncu --set full capture (B = 128)
    try:
        with open(os.path.join(REPO, "profiles", TRAFFIC_FILE)) as f:
            tr = json.load(f)["bytes"]
        knames = KERNEL_NAMES(B)[dom]
        kname = next((k for k in knames if k in tr), None)
        if B == 128 and nb == 1 and not args.real and kname is not None:
            roof["traffic"] = tr[kname]
            roof["traffic_source"] = f"profiles/{TRAFFIC_FILE} (dram__bytes_read.sum + dram__bytes_write.sum, ncu)"
    except (OSError, KeyError, ValueError):
        pass
    roof["timing"] = ("live: CUDA events around each stage launch inside the timed region" if live_profile else
                      "live: CUDA events around each stage launch (eager launches) in a second timed pass of "
                      "the same steps, right after the headline pass")
    t_roof = rscale * nb * wl.roofline_time(B, FP64_PEAK_TFLOPS * 1e12, peaks["hbm_gbs"] * 1e9)
    whole = 2 * wl.f_fwd(B) * nb / (ms * 1e-3) / 1e12

    line = {
        "metric": f"fwd+inv SGL transforms/s at B={B} fp64", "value": value, "unit": "transforms/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: coefficients with the config's BASELINE.json distribution (numpy PCG64, seed = rank)",
        "config": workload_config(B, nb, args.real),
        "setup": {"parallelism": f"replicas x{world}" if world > 1 else "single",
                  "batch_per_gpu": nb,
                  "path": "real fast path (sglgpu_*_real)" if args.real else "complex path (sglgpu_forward/inverse)",
                  "l2": f"inputs rotated over {nrot} coefficient buffers ({nrot * 16 * Om * nb / 1e6:.0f} MB) "
                        f"and every step writes/reads a {(8 if args.real else 16) * Ps * nb / 2**20:.0f} MiB grid "
                        "(> 126 MB L2)"},
        "e2e": {"value": world * nb / (e2e_ms / 1000.0), "unit": "transforms/s",
                "h2d_bytes_per_step": (16 * Om + (8 if args.real else 16) * Ps) * nb,
                "d2h_bytes_per_step": ((8 if args.real else 16) * Ps + 16 * Om) * nb,
                "ms_per_step": e2e_ms, "callers": callers,
                "single_caller_value": world * nb / (e2e_single_ms / 1000.0),
                "api": "paper_1604_05140_b200.ifsglft_batch/fsglft_batch (C ABI, pinned host memory; odd callers forward-first; "
                       f"{callers} concurrent host threads on one plan, each step's copies inside the timed region)"},
        "gpu_launches": gpu_launches,
        "roofline": roof,
        "transform_fp64_tflops": rscale * whole,
        "transform_roofline": {"per_stage_roofline_ms": 1e3 * t_roof, "measured_ms": ms, "frac": 1e3 * t_roof / ms,
                               "definition": "sum over both directions of max(F_s/P_fp64, Q_s/BW_hbm) for the "
                                             "spherical and radial stages (SURVEY.md 8(d))"},
        "stages": stage_info,
        "clocks": clk.summary(),
        "roundtrip_normwise_err": max(err, e2e_err),
    }
    if not (line["roundtrip_normwise_err"] < 1e-10):
        raise SystemExit(f"bench: round trip failed (normwise error {line['roundtrip_normwise_err']:.3e}); "
                         "refusing to report a timing of wrong results")
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference(B, nb, args.real, budget_s=15.0)
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

    # ---- exchange accounting (this rank): bytes it sends to peers per step and
    # the device time of the phases that carry them (a second pass of the same
    # steps with CUDA events between the phases; max over ranks)
    import paper_1604_05140_b200.distributed as D

    s0r, _ = part.shell_range(rank)
    nu0, nu1 = part.nu_range(rank)
    row = 16 * nb * sc  # bytes of one nu row of this rank's shells
    s_bytes = sum((part.nu_range(q)[1] - part.nu_range(q)[0]) * row for q in range(world) if q != rank)
    l0r, l1r = part.l_ranges[rank]
    omega_r = sum((2 * l + 1) * (B - l) for l in range(l0r, l1r))  # this rank's coefficients
    exch = {"forward_shell_rows_bytes": s_bytes, "inverse_shell_rows_bytes": s_bytes}
    if exchange == "fused":
        exch["forward_coefficients_bytes"] = 16 * nb * omega_r * (world - 1)  # peer stores of its degrees
    else:
        exch["forward_coefficients_bytes"] = 16 * nb * Om  # all_reduce payload
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    phase = np.zeros(6)
    dist.barrier()
    for s_ in range(args.steps):
        c = cin[s_ % nrot]
        evs[0].record(stream)
        if exchange == "fused":
            D.fused_inverse_radial(c, part, st, peers, rank)                    # radial inv + peer stores
            evs[1].record(stream)
            D._stream_barrier(dist, None, c.device)
            evs[2].record(stream)
            loc = D.fused_inverse_spherical(part, st, peers, rank, c.device)
            D._stream_barrier(dist, None, c.device)
            evs[3].record(stream)
            D.fused_forward_spherical(loc.view(nb, -1), part, st, peers, rank, nb)  # spherical fwd + peer stores
            evs[4].record(stream)
            D._stream_barrier(dist, None, c.device)
            evs[5].record(stream)
            if world > 1:
                D.fused_forward_radial_bcast(part, st, peers, rank, stream.cuda_stream)
                D._stream_barrier(dist, None, c.device)
            else:
                co = torch.zeros((nb, Om), dtype=torch.complex128, device="cuda")
                D.fused_forward_radial(part, st, peers, rank, co)
            evs[6].record(stream)
        else:
            l0, l1 = part.l_ranges[rank]
            blocks = st.radial_inverse(c, l0, l1, sc, nb) if l1 > l0 else torch.empty(0, dtype=torch.complex128,
                                                                                       device="cuda")
            evs[1].record(stream)
            recv = [(part.nu_range(q)[1] - part.nu_range(q)[0]) * nb * sc for q in range(world)]
            S_loc = D._a2a(dist, None, blocks, [(nu1 - nu0) * nb * sc] * world, recv)
            evs[2].record(stream)
            loc = st.spherical_inverse(S_loc, s0r, sc, nb)
            S_f = st.spherical_forward(loc.view(nb, -1), s0r, sc, nb)
            evs[3].record(stream)
            blk = D._a2a(dist, None, S_f, recv, [(nu1 - nu0) * nb * sc] * world)
            evs[4].record(stream)
            co = torch.zeros((nb, Om), dtype=torch.complex128, device="cuda")
            if l1 > l0:
                st.radial_forward(blk, l0, l1, sc, nb, co)
            evs[5].record(stream)
            dist.all_reduce(torch.view_as_real(co))
            evs[6].record(stream)
        torch.cuda.synchronize()
        for i in range(6):
            phase[i] += evs[i].elapsed_time(evs[i + 1])
    phase /= args.steps
    tph = torch.tensor(phase, device="cuda", dtype=torch.float64)
    dist.all_reduce(tph, op=dist.ReduceOp.MAX)
    phase = tph.cpu().numpy()
    names = (["radial_inverse+peer_stores", "barrier", "spherical_inverse(+barrier)", "spherical_forward+peer_stores",
              "barrier", "radial_forward+coefficient_peer_stores(+barrier)"] if exchange == "fused" else
             ["radial_inverse", "all_to_all(shells)", "spherical_inverse+spherical_forward", "all_to_all(shells)",
              "radial_forward", "all_reduce(coefficients)"])
    exch["phase_ms_max_over_ranks"] = {n: round(float(v), 5) for n, v in zip(names, phase)}
    exch["phase_sum_ms"] = round(float(phase.sum()), 5)

    line = {
        "metric": f"fwd+inv SGL transforms/s at B={B} fp64", "value": value, "unit": "transforms/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: iid complex normal coefficients (numpy PCG64, seed 0)",
        "config": workload_config(B, nb, False),
        "setup": {"split": f"{nb} function(s) per step split over {world} GPUs (shells / degree ranges, " +
                           ("exchange fused into the stage epilogues: NVLink peer stores" if exchange == "fused"
                            else "NCCL all-to-all") + ")",
                  "exchange": exchange + (f" ({why})" if why else ""),
                  "parallelism": f"shell/(l,m) split x{world}",
                  "l2": f"inputs rotated over {nrot} buffers; per-step grid {16 * Ps * nb / 2**20:.0f} MiB > L2"},
        "exchange": exch,
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
