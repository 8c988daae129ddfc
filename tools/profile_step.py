"""Small driver for ncu: B round trips (inverse + forward) at bandlimit B on cuda:0."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_05140_b200 as sgl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=128)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
plan = sgl.TransformPlan.compute(a.B, device=0)
n = sgl.coefficient_count(a.B)
rng = np.random.default_rng(0)
c = torch.from_numpy((rng.standard_normal((a.batch, n)) + 1j * rng.standard_normal((a.batch, n))) / 2 ** 0.5).cuda()
for _ in range(a.steps):
    g = sgl.ifsglft_batch(plan, c)
    b = sgl.fsglft_batch(plan, g)
torch.cuda.synchronize()
err = float((b - c).abs().max() / c.abs().max())
print(f"B={a.B} batch={a.batch} roundtrip err {err:.2e}")
assert err < 1e-11
