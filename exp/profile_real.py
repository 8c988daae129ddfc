"""ncu driver: real-valued round trips (config C5 shape) on cuda:0."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1604_05140_b200 as sgl
B = int(os.environ.get("B", 32)); nb = int(os.environ.get("NB", 4096)); steps = int(os.environ.get("STEPS", 2))
plan = sgl.TransformPlan.compute(B, device=0)
c = torch.randn(nb, sgl.coefficient_count(B), dtype=torch.complex128, device="cuda")
for _ in range(steps):
    x = sgl.ifsglft_real_batch(plan, c)
    b = sgl.fsglft_real_batch(plan, x)
torch.cuda.synchronize()
print("ok", x.shape)
