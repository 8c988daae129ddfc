"""The multi-GPU shell / (l, m) decomposition (paper_1604_05140_b200.distributed)
run as world_size 2 and 4 over gloo on CPU, with the oracle's stage functions
standing in for the CUDA stages.  The distributed forward / inverse must equal
the single-process oracle transform."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1604_05140_b200.distributed import Partition, fsglft_distributed, ifsglft_distributed


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, B, batch, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from device_model import ModelStages
        from oracle_bindings import Oracle, coefficient_count, sample_count

        part = Partition.make(B, world)
        stages = ModelStages(B)
        orc = Oracle(B)
        rng = np.random.default_rng(7)
        c = (rng.standard_normal((batch, coefficient_count(B))) + 1j * rng.standard_normal((batch, coefficient_count(B))))
        g_full = np.stack([orc.inverse(c[f]) for f in range(batch)])
        s0, s1 = part.shell_range(rank)
        n_sh = 4 * B * B
        g_local = torch.from_numpy(np.ascontiguousarray(g_full[:, s0 * n_sh:s1 * n_sh]))
        coeffs = fsglft_distributed(g_local, part, stages, dist, batch=batch).numpy()
        ref = np.stack([orc.forward(g_full[f]) for f in range(batch)])
        e_fwd = float(np.abs(coeffs - ref).max() / np.abs(ref).max())
        g_back = ifsglft_distributed(torch.from_numpy(c), part, stages, dist, batch=batch).numpy().reshape(batch, -1)
        e_inv = float(np.abs(g_back - g_full[:, s0 * n_sh:s1 * n_sh]).max() / np.abs(g_full).max())
        q.put((rank, e_fwd, e_inv))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,B,batch", [(2, 4, 1), (2, 8, 2), (4, 8, 1)])
def test_distributed_matches_single_process(world, B, batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = [q.get(timeout=10) for _ in range(world)]
    for rank, e_fwd, e_inv in res:
        assert e_fwd < 1e-13 and e_inv < 1e-13, (rank, e_fwd, e_inv)


def test_partition_balances_radial_work():
    for B, W in ((128, 8), (256, 8), (64, 2), (16, 4)):
        p = Partition.make(B, W)
        assert p.l_ranges[0][0] == 0 and p.l_ranges[-1][1] == B
        assert all(a[1] == b[0] for a, b in zip(p.l_ranges, p.l_ranges[1:]))
        work = [sum((2 * l + 1) * (B - l) for l in range(*lr)) for lr in p.l_ranges]
        assert max(work) <= 1.25 * sum(work) / W + (2 * B) * B
        assert p.shells_per_rank * W == 2 * B
    with pytest.raises(ValueError):
        Partition.make(3, 4)


def test_peer_buffer_layout_matches_radial_blocks():
    """The fused exchange's destinations (PeerBuffers.fwd_dst) place source rank r's
    shell block where sglgpu_radial_forward reads block r of the owner's receive
    buffer: [src][nu - nu0_q][f][i_local], blk_stride = (nu1 - nu0) * row."""
    from paper_1604_05140_b200.distributed import PeerBuffers

    B, W, batch = 16, 4, 3
    part = Partition.make(B, W)
    row = batch * part.shells_per_rank
    fwd = [(1 << 40) + (q << 32) for q in range(W)]  # fake device addresses
    peers = PeerBuffers(part, batch, fwd, [0] * W, [], [])
    for r in range(W):
        dst = list(peers.fwd_dst(r))
        for q in range(W):
            nu0, nu1 = part.nu_range(q)
            assert dst[q] == fwd[q] + r * (nu1 - nu0) * row * 16
    for q in range(W):
        fb, ib = PeerBuffers.sizes(part, batch, q)
        nu0, nu1 = part.nu_range(q)
        assert fb == W * (nu1 - nu0) * row * 16 and ib == B * B * row * 16
