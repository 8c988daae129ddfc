"""Phase clocks of the INT8 Legendre inverse (SGL_I8_TRACE = device buffer address)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
B = int(os.environ.get("B", 128))
buf = torch.zeros(20000 * 64, dtype=torch.int64, device="cuda")
os.environ["SGL_I8"] = "leginv"
os.environ["SGL_I8_TRACE"] = str(buf.data_ptr())
import paper_1604_05140_b200 as sgl
plan = sgl.TransformPlan.compute(B, device=0)
n = sgl.coefficient_count(B)
c = torch.randn(1, n, dtype=torch.complex128, device="cuda")
for _ in range(3):
    g = sgl.ifsglft_batch(plan, c)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(-1, 8, 8)
t = t[t[:, 0, 0] != 0]
names = ["load+max", "digits+alloc+sync", "mma issue", "mma wait", "epi first tmem ld", "epi rest", "sync+dealloc"]
d = []
for tile in range(8):
    x = t[:, tile, [0, 1, 2, 3, 4, 7, 5, 6]]
    ok = (x != 0).all(axis=1)
    if ok.sum() == 0: continue
    d.append(np.diff(x[ok], axis=1))
d = np.concatenate(d)
print(f"B={B} units {t.shape[0]} tiles {d.shape[0]}  mean cycles per phase:")
for i, nm in enumerate(names): print(f"  {nm:22s} {d[:, i].mean():8.0f}  (p50 {np.median(d[:, i]):.0f}, p90 {np.percentile(d[:, i], 90):.0f})")
print("  total per tile", d.sum(axis=1).mean())
