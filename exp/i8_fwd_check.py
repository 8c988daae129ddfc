"""INT8 tensor-core Legendre forward (SGL_I8=legfwd) vs the DMMA path and the CPU oracle."""
import os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_1604_05140_b200 as sgl
from oracle_bindings import Oracle, normwise
for B in [int(x) for x in sys.argv[1:]] or [32, 64, 128]:
    plan = sgl.TransformPlan.compute(B, device=0)
    rng = np.random.default_rng(B)
    n = sgl.coefficient_count(B)
    c = (rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n))) / np.sqrt(2)
    ct = torch.tensor(c, dtype=torch.complex128, device="cuda")
    os.environ["SGL_I8"] = "0"
    g = sgl.ifsglft_batch(plan, ct)
    f0 = sgl.fsglft_batch(plan, g).cpu().numpy()
    for nb in (1, 2):
        os.environ["SGL_I8"] = "legfwd"
        f1 = sgl.fsglft_batch(plan, g[:nb].contiguous()).cpu().numpy()
        os.environ["SGL_I8"] = "0"
        msg = f"B={B} nb={nb}: i8 vs dmma {max(normwise(f1[b], f0[b]) for b in range(nb)):.2e} vs coeffs {max(normwise(f1[b], c[b]) for b in range(nb)):.2e} finite {np.isfinite(f1).all()}"
        if B <= 64:
            orc = Oracle(B)
            msg += f" vs oracle {normwise(f1[0], orc.forward(g[0].cpu().numpy())):.2e}"
        print(msg, flush=True)
