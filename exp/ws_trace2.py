"""Event clocks of the warp-specialised INT8 Legendre inverse (8 tiles x 8 events)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
B = int(os.environ.get("B", 128))
buf = torch.zeros(4000 * 64, dtype=torch.int64, device="cuda")
os.environ["SGL_I8"] = "ws"
os.environ["SGL_I8_TRACE"] = str(buf.data_ptr())
import paper_1604_05140_b200 as sgl
plan = sgl.TransformPlan.compute(B, device=0)
c = torch.randn(1, sgl.coefficient_count(B), dtype=torch.complex128, device="cuda")
for _ in range(3): g = sgl.ifsglft_batch(plan, c)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(-1, 8, 8)
t = t[(t[:, :, 0] != 0).all(axis=1)]
rel = t - t[:, 0:1, 0:1]
names = ["P cp.async done", "P data_empty ok", "P max done", "P arrive full", "M full ok", "M tmem_empty ok", "M issued", "E got"]
print("units", t.shape[0])
print("tile " + " ".join(f"{n:>16s}" for n in names))
for i in range(8):
    print(f"{i:4d} " + " ".join(f"{rel[:, i, e].mean():16.0f}" for e in range(8)))
