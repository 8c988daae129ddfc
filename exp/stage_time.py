"""Stage times of B round trips without a correctness check (for timing-only variants)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1604_05140_b200 as sgl
B = int(os.environ.get("B", 128)); steps = int(os.environ.get("STEPS", 50))
plan = sgl.TransformPlan.compute(B, device=0)
L = sgl.lib()
n = sgl.coefficient_count(B)
c = torch.randn(int(os.environ.get("BATCH", 1)), n, dtype=torch.complex128, device="cuda")
g = sgl.ifsglft_batch(plan, c); b = sgl.fsglft_batch(plan, g)
ms = np.zeros(8); cnt = np.zeros(8, dtype=np.int32)
assert L.sglgpu_profile_begin(plan.handle) == 0
for _ in range(steps):
    sgl.ifsglft_batch(plan, c, out=g); sgl.fsglft_batch(plan, g, out=b)
torch.cuda.synchronize()
assert L.sglgpu_profile_end(plan.handle, ms.ctypes.data, cnt.ctypes.data) == 0
names = ["az_fwd", "leg_fwd", "rad_fwd", "rad_inv", "leg_inv", "az_inv", "sph_fwd", "sph_inv"]
print(os.environ.get("SGL_B200_LIB", "default"), " ".join(f"{nm}={ms[i] / max(cnt[i], 1) * 1e3:.1f}" for i, nm in enumerate(names)))
