"""Command-line front end with the reference's record formats.

    python -m paper_1604_05140_b200.cli roundtrip --bandlimit 64 --repetitions 10 [--csv out.csv]
    python -m paper_1604_05140_b200.cli bench --bandlimits 2,4,8,16,32 [--repetitions 10] [--csv out.csv]
    python -m paper_1604_05140_b200.cli transform --direction fwd|inv --bandlimit B --in X --out Y

Mirrors `sglfft roundtrip|bench|transform` (tools/main.cpp:13-116,
tools/commands.cpp): the same coefficient stream (mt19937_64, top-53-bit map to
[-1, 1), commands.cpp:73-88), the same timed region (one inverse + one forward,
plan excluded, commands.cpp:152-177), the same table / CSV row formats
(`B,variant,reps,mean_time_s,mean_max_abs_err,mean_max_rel_err`,
commands.hpp:17-32, commands.cpp:18-71, 179-192) and the same raw vector files
(interleaved f64 LE, commands.cpp:194-226).  Only the `fast` variant exists here
(the naive O(B^7) / separated O(B^6) rungs are reference oracles, not GPU code).
Exit codes: 0 ok, 1 runtime error, 2 usage error (main.cpp:84-91).
Tables: --tables DIR, else $SGL_TABLES, else the packaged radial rules
(acquire_plan, commands.cpp:90-114).
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

CSV_HEADER = "B,variant,reps,mean_time_s,mean_max_abs_err,mean_max_rel_err"


class MT19937_64:
    """std::mt19937_64, vectorized twist (numpy uint64)."""

    N, M = 312, 156
    A = np.uint64(0xB5026F5AA96619E9)
    UM, LM = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [seed & 0xFFFFFFFFFFFFFFFF]
        for i in range(1, self.N):
            prev = mt[-1]
            mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
        self.mt = np.array(mt, dtype=np.uint64)
        self.idx = self.N

    def _twist(self):
        mt = self.mt
        N, M = self.N, self.M
        one = np.uint64(1)
        # same element order as the scalar algorithm: i < N-M uses old values at i+M;
        # i >= N-M uses the already updated ones (wraps to the front)
        for lo, hi in ((0, N - M), (N - M, N - 1)):
            i = np.arange(lo, hi)
            x = (mt[i] & self.UM) | (mt[i + 1] & self.LM)
            y = (x >> one) ^ np.where(x & one, self.A, np.uint64(0))
            mt[i] = mt[(i + M) % N] ^ y
        x = (mt[N - 1] & self.UM) | (mt[0] & self.LM)
        mt[N - 1] = mt[M - 1] ^ (x >> one) ^ (self.A if int(x) & 1 else np.uint64(0))
        self.idx = 0

    def next(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        got = 0
        while got < n:
            if self.idx >= self.N:
                self._twist()
            take = min(n - got, self.N - self.idx)
            x = self.mt[self.idx:self.idx + take].copy()
            x ^= (x >> np.uint64(29)) & np.uint64(0x5555555555555555)
            x ^= (x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
            x ^= (x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
            x ^= x >> np.uint64(43)
            out[got:got + take] = x
            got += take
            self.idx += take
        return out


class CoefficientStream:
    """commands.cpp:73-88: real then imaginary part, 2 * ((x >> 11) * 2^-53) - 1."""

    def __init__(self, seed: int):
        self.engine = MT19937_64(seed)

    def next(self, B: int) -> np.ndarray:
        import paper_1604_05140_b200 as sgl

        n = sgl.coefficient_count(B)
        x = self.engine.next(2 * n)
        d = 2.0 * ((x >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)) - 1.0
        return d.view(np.complex128)


def _plan(B: int, tables: str | None):
    import paper_1604_05140_b200 as sgl

    d = tables or os.environ.get("SGL_TABLES")
    if d:
        return sgl.TransformPlan.from_tables(d, B)
    return sgl.TransformPlan.compute(B)


def run_roundtrip(B, repetitions, seed, tables=None):
    import paper_1604_05140_b200 as sgl

    if repetitions < 1:
        raise RuntimeError("repetitions must be at least 1")
    plan = _plan(B, tables)
    stream = CoefficientStream(seed)
    # plan creation / table upload outside the timed region
    plan.handle
    t_sum = a_sum = r_sum = 0.0
    for _ in range(repetitions):
        c = stream.next(B)
        t0 = time.perf_counter()
        g = sgl.ifsglft(sgl.SglCoefficients(B, c), plan)
        back = sgl.fsglft(g, plan)
        t1 = time.perf_counter()
        e = sgl.roundtrip_error(c, back.values)
        if e.nonfinite:
            raise RuntimeError(f"non-finite output at B = {B}")
        t_sum += t1 - t0
        a_sum += e.max_abs
        r_sum += e.max_rel
    return dict(B=B, variant="fast", reps=repetitions, mean_time_s=t_sum / repetitions,
                mean_max_abs_err=a_sum / repetitions, mean_max_rel_err=r_sum / repetitions)


def header_line() -> str:
    return "%4s  %-9s  %4s  %12s  %13s  %13s" % ("B", "variant", "reps", "mean_time_s", "mean_max_abs",
                                               "mean_max_rel")


def record_line(r) -> str:
    return "%4d  %-9s  %4d  %12.6f  %13.6e  %13.6e" % (r["B"], r["variant"], r["reps"], r["mean_time_s"],
                                                     r["mean_max_abs_err"], r["mean_max_rel_err"])


def csv_line(r) -> str:
    return "%d,%s,%d,%.17g,%.17g,%.17g" % (r["B"], r["variant"], r["reps"], r["mean_time_s"],
                                          r["mean_max_abs_err"], r["mean_max_rel_err"])


def append_csv(path, records):
    fresh = not os.path.exists(path) or os.path.getsize(path) == 0
    with open(path, "a") as f:
        if fresh:
            f.write(CSV_HEADER + "\n")
        for r in records:
            f.write(csv_line(r) + "\n")


def read_csv(path):
    out = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line or line == CSV_HEADER:
                continue
            B, variant, reps, t, a, r = line.split(",")
            out.append(dict(B=int(B), variant=variant, reps=int(reps), mean_time_s=float(t),
                            mean_max_abs_err=float(a), mean_max_rel_err=float(r)))
    return out


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="sglfft-b200", description="Spherical Gauss-Laguerre Fourier transforms (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    rt = sub.add_parser("roundtrip", help="Inverse+forward roundtrip on random coefficients")
    rt.add_argument("--bandlimit", type=int, required=True)
    rt.add_argument("--variant", default="fast", choices=["fast"])
    rt.add_argument("--repetitions", type=int, default=10)
    rt.add_argument("--seed", type=int, default=0)
    rt.add_argument("--threads", type=int, default=0, help="accepted for compatibility; ignored")
    rt.add_argument("--csv")
    rt.add_argument("--tables")
    be = sub.add_parser("bench", help="Roundtrip benchmark over bandlimits")
    be.add_argument("--bandlimits", default="2,4,8,16,32")
    be.add_argument("--variants", default="fast")
    be.add_argument("--repetitions", type=int, default=10)
    be.add_argument("--seed", type=int, default=0)
    be.add_argument("--threads", type=int, default=0)
    be.add_argument("--csv")
    be.add_argument("--tables")
    tr = sub.add_parser("transform", help="Transform a raw complex vector file")
    tr.add_argument("--direction", required=True, choices=["fwd", "inv"])
    tr.add_argument("--bandlimit", type=int, required=True)
    tr.add_argument("--in", dest="inp", required=True)
    tr.add_argument("--out", required=True)
    tr.add_argument("--variant", default="fast", choices=["fast"])
    tr.add_argument("--threads", type=int, default=0)
    tr.add_argument("--tables")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        import paper_1604_05140_b200 as sgl

        if args.cmd == "roundtrip":
            rec = run_roundtrip(args.bandlimit, args.repetitions, args.seed, args.tables)
            print(f"# device: B200 (sm_100a), seed: {args.seed}")
            print(header_line())
            print(record_line(rec))
            if args.csv:
                append_csv(args.csv, [rec])
        elif args.cmd == "bench":
            variants = args.variants.split(",")
            if any(v != "fast" for v in variants):
                raise ValueError("only the fast variant runs on the GPU")
            print(f"# device: B200 (sm_100a), seed: {args.seed}")
            print(header_line())
            recs = []
            for B in (int(b) for b in args.bandlimits.split(",")):
                recs.append(run_roundtrip(B, args.repetitions, args.seed, args.tables))
                print(record_line(recs[-1]))
            if args.csv:
                append_csv(args.csv, recs)
        else:
            B = args.bandlimit
            plan = _plan(B, args.tables)
            n_in = sgl.sample_count(B) if args.direction == "fwd" else sgl.coefficient_count(B)
            size = os.path.getsize(args.inp)
            if size != 16 * n_in:
                raise RuntimeError(f"input vector {args.inp} holds {size // 16} complex values, expected {n_in}")
            x = np.fromfile(args.inp, dtype="<f8").view(np.complex128)
            if args.direction == "fwd":
                y = sgl.fsglft(sgl.SampleGrid(B, x), plan).values
            else:
                y = sgl.ifsglft(sgl.SglCoefficients(B, x), plan).values
            np.ascontiguousarray(y, dtype=np.complex128).view("<f8").tofile(args.out)
        return 0
    except Exception as e:  # noqa: BLE001 -- mirrors the reference's catch-all (commands.cpp:235-238)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
