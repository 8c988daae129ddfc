"""torchrun helper for tests/test_gpu_parity.py::test_fused_exchange_ipc_two_processes:
the fused exchange (NVLink peer stores into CUDA-IPC-mapped receive buffers) with
two processes.  On the one-GPU test box both processes share cuda:0 -- the IPC
mapping, the peer-store epilogues and the buffer layouts are exercised; the
ranks synchronize through CPU barriers (gloo), no kernel waits on another rank."""
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
from paper_1604_05140_b200.distributed import (CudaStages, Partition, PeerBuffers, fused_forward_radial,  # noqa: E402
                                               fused_forward_radial_bcast, fused_forward_spherical,
                                               fused_inverse_radial, fused_inverse_spherical)


def cpu_barrier():
    torch.cuda.synchronize()
    dist.barrier()


def main():
    dev = int(os.environ.get("SGL_FUSED_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    B, nb = int(sys.argv[1]), int(sys.argv[2])
    r, w = dist.get_rank(), dist.get_world_size()
    plan = sgl.TransformPlan.compute(B, device=dev)
    part = Partition.make(B, w)
    st = CudaStages(plan)
    peers = PeerBuffers.exchange(part, nb, dist)
    orc = Oracle(B)
    rng = np.random.default_rng(5)
    n = sgl.coefficient_count(B)
    c = (rng.standard_normal((nb, n)) + 1j * rng.standard_normal((nb, n))) / np.sqrt(2)
    dc = torch.from_numpy(c).cuda()
    # inverse: radial stage stores shell blocks into the owners' S buffers
    fused_inverse_radial(dc, part, st, peers, r)
    cpu_barrier()
    loc = fused_inverse_spherical(part, st, peers, r, dc.device).view(nb, -1)
    # forward: spherical stage stores S rows into the owners' receive buffers
    fused_forward_spherical(loc.contiguous(), part, st, peers, r, nb)
    cpu_barrier()
    coeffs = torch.zeros((nb, n), dtype=torch.complex128, device=dc.device)
    fused_forward_radial(part, st, peers, r, coeffs)
    torch.cuda.synchronize()
    back = torch.view_as_real(coeffs).cpu()
    dist.all_reduce(back)  # disjoint degree ranges: the sum assembles the vector
    back = torch.view_as_complex(back).numpy()
    # the fused assembly: every rank's radial epilogue stores its degrees into all
    # ranks' (IPC-mapped) coefficient vectors
    fused_forward_radial_bcast(part, st, peers, r)
    cpu_barrier()
    mine = peers.coef_tensor(r).cpu().numpy()
    s0, s1 = part.shell_range(r)
    nsh = 4 * B * B
    loc = loc.cpu().numpy()
    for f in range(nb):
        g_ref = orc.inverse(c[f])[s0 * nsh:s1 * nsh]
        assert normwise(loc[f], g_ref) < 1e-12, normwise(loc[f], g_ref)
        assert normwise(back[f], c[f]) < 1e-12, normwise(back[f], c[f])
        assert np.array_equal(mine[f], back[f]), "broadcast assembly differs from the all-reduce"
    cpu_barrier()
    peers.close()
    if r == 0:
        print("fused exchange OK")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
