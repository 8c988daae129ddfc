"""Small driver for compute-sanitizer: complex and real paths, several bandlimits
(pow2 FFT kernels, the naive non-pow2 kernels), batch > 1, stage entry points."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_05140_b200 as sgl  # noqa: E402
from paper_1604_05140_b200.distributed import CudaStages, Partition  # noqa: E402

rng = np.random.default_rng(0)
for B, nb in ((3, 2), (8, 3), (16, 1), (32, 2)):
    plan = sgl.TransformPlan.compute(B, device=0)
    n = sgl.coefficient_count(B)
    c = torch.from_numpy(rng.standard_normal((nb, n)) + 1j * rng.standard_normal((nb, n))).cuda()
    g = sgl.ifsglft_batch(plan, c)
    b = sgl.fsglft_batch(plan, g)
    if B >= 2 and (2 * B) & (2 * B - 1) == 0:
        gr = sgl.ifsglft_real_batch(plan, c)
        sgl.fsglft_real_batch(plan, gr)
        st = CudaStages(plan)
        part = Partition.make(B, 2)
        S = st.spherical_forward(g[:, :part.shells_per_rank * 4 * B * B].contiguous(), 0, part.shells_per_rank, nb)
    torch.cuda.synchronize()
    print(B, float((b - c).abs().max() / c.abs().max()))
