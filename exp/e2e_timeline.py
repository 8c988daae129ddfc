"""Per-call host timeline of two anti-phase round-trip callers."""
import os, sys, threading, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1604_05140_b200 as sgl
B = int(os.environ.get("B", 128)); n = sgl.coefficient_count(B); P = sgl.sample_count(B)
plan = sgl.TransformPlan.compute(B, device=0)
pin = lambda shape: torch.empty(shape, dtype=torch.complex128).pin_memory().numpy()
bufs = []
for i in range(2):
    hc, hg, hb = pin((1, n)), pin((1, P)), pin((1, n))
    hc[:] = np.random.default_rng(i).standard_normal(n)
    sgl.ifsglft_batch(plan, hc, out=hg); sgl.fsglft_batch(plan, hg, out=hb)
    sgl.ifsglft_batch(plan, hc, out=hg); sgl.fsglft_batch(plan, hg, out=hb)
    bufs.append((hc, hg, hb))
log = []
T0 = time.perf_counter()
def w(i):
    hc, hg, hb = bufs[i]
    for k in range(4):
        for d in ((0, 1) if i == 0 else (1, 0)):
            t = time.perf_counter()
            if d == 0: sgl.ifsglft_batch(plan, hc, out=hg)
            else: sgl.fsglft_batch(plan, hg, out=hb)
            log.append((i, "inv" if d == 0 else "fwd", (t - T0) * 1e3, (time.perf_counter() - T0) * 1e3))
ts = [threading.Thread(target=w, args=(i,)) for i in range(2)]
[x.start() for x in ts]; [x.join() for x in ts]
for r in sorted(log, key=lambda r: r[2]): print(f"caller {r[0]} {r[1]}  {r[2]:7.2f} -> {r[3]:7.2f}  ({r[3]-r[2]:5.2f} ms)")
