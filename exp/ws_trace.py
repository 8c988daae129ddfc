"""Role clocks of the warp-specialised INT8 Legendre inverse: per tile, producer done (0),
MMAs issued (1), epilogue got TMEM (3), epilogue released TMEM (2)."""
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
t = buf.cpu().numpy().reshape(-1, 16, 4)
t = t[(t[:, :, 0] != 0).all(axis=1)]
t0 = t[:, :1, 0:1]
rel = t - t[:, 0:1, 0:1]
print("units", t.shape[0], " mean clock (relative to producer tile 0 done) per tile: prod, mma, epi-got, epi-released")
for i in range(16):
    print(i, " ".join(f"{rel[:, i, r].mean():9.0f}" for r in (0, 1, 3, 2)))
d = np.diff(rel[:, :, 2], axis=1).mean()
print("epilogue release interval", d, " producer interval", np.diff(rel[:, :, 0], axis=1).mean(), " mma interval", np.diff(rel[:, :, 1], axis=1).mean())
