"""Host-API duplex check: one thread only ifsglft (big D2H), another only fsglft (big H2D)."""
import os, sys, threading, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1604_05140_b200 as sgl
B = int(os.environ.get("B", 128)); n = sgl.coefficient_count(B); P = sgl.sample_count(B)
plan = sgl.TransformPlan.compute(B, device=0)
pin = lambda shape: torch.empty(shape, dtype=torch.complex128).pin_memory().numpy()
hc, hg, hb, hg2 = pin((1, n)), pin((1, P)), pin((1, n)), pin((1, P))
hc[:] = (np.random.default_rng(0).standard_normal(n) + 0j)
sgl.ifsglft_batch(plan, hc, out=hg); sgl.fsglft_batch(plan, hg, out=hb); sgl.ifsglft_batch(plan, hc, out=hg2)
K = 8
def inv_loop():
    for _ in range(K): sgl.ifsglft_batch(plan, hc, out=hg2)
def fwd_loop():
    for _ in range(K): sgl.fsglft_batch(plan, hg, out=hb)
for name, fns in [("inv alone", [inv_loop]), ("fwd alone", [fwd_loop]), ("inv || fwd", [inv_loop, fwd_loop]),
                  ("inv || inv", [inv_loop, inv_loop])]:
    t = time.perf_counter(); ts = [threading.Thread(target=f) for f in fns]
    [x.start() for x in ts]; [x.join() for x in ts]
    dt = time.perf_counter() - t
    print(f"{name:12s} {dt / K * 1e3:7.2f} ms per loop iteration ({len(fns)} thread(s))")
def rt_a():
    for _ in range(K // 2): sgl.ifsglft_batch(plan, hc, out=hg); sgl.fsglft_batch(plan, hg, out=hb)
hg3, hb3, hc3 = pin((1, P)), pin((1, n)), pin((1, n))
hg3[:] = hg
def rt_b():
    for _ in range(K // 2): sgl.fsglft_batch(plan, hg3, out=hb3); sgl.ifsglft_batch(plan, hb3, out=hg3)
for name, fns in [("rt A alone", [rt_a]), ("rt A || rt B", [rt_a, rt_b]), ("rt A || rt A'", [rt_a, rt_b])]:
    t = time.perf_counter(); ts = [threading.Thread(target=f) for f in fns]
    [x.start() for x in ts]; [x.join() for x in ts]
    dt = time.perf_counter() - t
    print(f"{name:14s} {dt / (K // 2) * 1e3:7.2f} ms per round trip per thread ({len(fns)} thread(s))")
