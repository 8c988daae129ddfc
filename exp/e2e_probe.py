"""Per-call timing of host-memory transforms (pinned numpy buffers) at B=128."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1604_05140_b200 as sgl
B = int(os.environ.get("B", 128)); nb = int(os.environ.get("NB", 1))
plan = sgl.TransformPlan.compute(B, device=0)
Om, Ps = sgl.coefficient_count(B), sgl.sample_count(B)
hc = torch.empty((nb, Om), dtype=torch.complex128).pin_memory().numpy(); hc[:] = 1.0
hg = torch.empty((nb, Ps), dtype=torch.complex128).pin_memory().numpy()
hb = torch.empty((nb, Om), dtype=torch.complex128).pin_memory().numpy()
for _ in range(2):
    sgl.ifsglft_batch(plan, hc, out=hg); sgl.fsglft_batch(plan, hg, out=hb)
ti, tf = [], []
for _ in range(5):
    t0 = time.perf_counter(); sgl.ifsglft_batch(plan, hc, out=hg); t1 = time.perf_counter()
    sgl.fsglft_batch(plan, hg, out=hb); t2 = time.perf_counter()
    ti.append(t1 - t0); tf.append(t2 - t1)
# raw copies for reference
d = torch.empty((nb, Ps), dtype=torch.complex128, device="cuda")
hgt = torch.from_numpy(hg)
torch.cuda.synchronize()
t0 = time.perf_counter(); d.copy_(hgt); torch.cuda.synchronize(); t1 = time.perf_counter(); hgt.copy_(d); torch.cuda.synchronize(); t2 = time.perf_counter()
print(os.environ.get("SGL_HOST_SERIAL", "-"), f"inv {1e3*np.median(ti):.2f} ms  fwd {1e3*np.median(tf):.2f} ms  raw H2D {1e3*(t1-t0):.2f} D2H {1e3*(t2-t1):.2f} ms ({16*Ps*nb/1e6:.0f} MB)")
