"""Stage times of real-valued round trips (config C5 shape by default)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1604_05140_b200 as sgl
B = int(os.environ.get("B", 32)); nb = int(os.environ.get("NB", 4096)); steps = int(os.environ.get("STEPS", 5))
plan = sgl.TransformPlan.compute(B, device=0)
L = sgl.lib()
c = torch.randn(nb, sgl.coefficient_count(B), dtype=torch.complex128, device="cuda")
x = sgl.ifsglft_real_batch(plan, c); b = sgl.fsglft_real_batch(plan, x)
ms = np.zeros(8); cnt = np.zeros(8, dtype=np.int32)
assert L.sglgpu_profile_begin(plan.handle) == 0
for _ in range(steps):
    sgl.ifsglft_real_batch(plan, c, out=x); sgl.fsglft_real_batch(plan, x, out=b)
torch.cuda.synchronize()
assert L.sglgpu_profile_end(plan.handle, ms.ctypes.data, cnt.ctypes.data) == 0
names = ["az_fwd", "leg_fwd", "rad_fwd", "rad_inv", "leg_inv", "az_inv", "sph_fwd", "sph_inv"]
print(os.environ.get("SGL_B200_LIB", "default"), " ".join(f"{nm}={ms[i] / steps * 1e3:.1f}" for i, nm in enumerate(names)))
