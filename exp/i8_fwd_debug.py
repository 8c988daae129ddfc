import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1604_05140_b200 as sgl
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
plan = sgl.TransformPlan.compute(B, device=0)
n = sgl.coefficient_count(B)
rng = np.random.default_rng(1)
c = torch.tensor((rng.standard_normal((1, n)) + 1j * rng.standard_normal((1, n))), device="cuda")
os.environ["SGL_I8"] = "0"
g = sgl.ifsglft_batch(plan, c)
f0 = sgl.fsglft_batch(plan, g).cpu().numpy()[0]
os.environ["SGL_I8"] = "legfwd"
f1 = sgl.fsglft_batch(plan, g).cpu().numpy()[0]
bad = ~np.isfinite(f1)
print("nonfinite", bad.sum(), "of", f1.size)
idx = [(nn, l, m) for nn in range(1, B + 1) for l in range(nn) for m in range(-l, l + 1)]
err = np.abs(f1 - f0)
order = np.argsort(-np.nan_to_num(err, nan=1e300))[:10]
for o in order[:3]: print(idx[o], f0[o], f1[o])
ok = np.isfinite(f1)
print("max rel err on finite:", np.max(err[ok]) / np.max(np.abs(f0)))
ms = np.array([m for (nn, l, m) in idx]); ls = np.array([l for (nn, l, m) in idx])
rel = err / np.max(np.abs(f0))
for m in range(-B + 1, B):
    sel = ms == m
    if sel.any() and rel[sel].max() > 1e-10: print("m", m, "max rel", rel[sel].max(), "l with err:", sorted(set(ls[sel][rel[sel] > 1e-10]))[:12])
