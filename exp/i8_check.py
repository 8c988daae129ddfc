"""INT8 tensor-core Legendre inverse vs the DMMA path and the CPU oracle (timing-free check)."""
import os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_1604_05140_b200 as sgl
from oracle_bindings import Oracle, per_shell, normwise
Bs = [int(x) for x in sys.argv[1:]] or [8, 16, 32, 64, 128]
for B in Bs:
    plan = sgl.TransformPlan.compute(B, device=0)
    rng = np.random.default_rng(B)
    n = sgl.coefficient_count(B)
    c = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / np.sqrt(2)
    ct = torch.tensor(c, dtype=torch.complex128, device="cuda").reshape(1, n)
    os.environ["SGL_I8"] = "0"
    g0 = sgl.ifsglft_batch(plan, ct); torch.cuda.synchronize()
    os.environ["SGL_I8"] = os.environ.get("I8MODE", "leginv")
    t = time.time(); g1 = sgl.ifsglft_batch(plan, ct); torch.cuda.synchronize(); dt = time.time() - t
    a, b = g0.cpu().numpy().ravel(), g1.cpu().numpy().ravel()
    msg = f"B={B}: i8 vs dmma per-shell {per_shell(b, a, B):.2e} finite {np.isfinite(b).all()}"
    if B <= 64:
        msg += f"  vs oracle {per_shell(b, Oracle(B).inverse(c), B):.2e}"
    print(msg, f"({dt*1e3:.1f} ms first call)", flush=True)
