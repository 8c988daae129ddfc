"""torchrun helper for tests/test_gpu_parity.py::test_nccl_split_path: the
distributed shell / (l, m) path over NCCL (one rank per GPU) against the oracle."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import paper_1604_05140_b200 as sgl  # noqa: E402
from oracle_bindings import Oracle, normwise  # noqa: E402
from paper_1604_05140_b200.distributed import CudaStages, Partition, fsglft_distributed, ifsglft_distributed  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B, nb = int(sys.argv[1]), int(sys.argv[2])
    r, w = dist.get_rank(), dist.get_world_size()
    plan = sgl.TransformPlan.compute(B, device=local)
    part = Partition.make(B, w)
    st = CudaStages(plan)
    orc = Oracle(B)
    rng = np.random.default_rng(3)
    n = sgl.coefficient_count(B)
    c = (rng.standard_normal((nb, n)) + 1j * rng.standard_normal((nb, n))) / np.sqrt(2)
    loc = ifsglft_distributed(torch.from_numpy(c).cuda(), part, st, dist, batch=nb)
    back = fsglft_distributed(loc, part, st, dist, batch=nb).cpu().numpy()
    s0, s1 = part.shell_range(r)
    nsh = 4 * B * B
    loc = loc.view(nb, -1).cpu().numpy()
    for f in range(nb):
        g_ref = orc.inverse(c[f])[s0 * nsh:s1 * nsh]
        assert normwise(loc[f], g_ref) < 1e-12, normwise(loc[f], g_ref)
        assert normwise(back[f], c[f]) < 1e-12
    dist.barrier()
    if r == 0:
        print("NCCL split path OK")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
