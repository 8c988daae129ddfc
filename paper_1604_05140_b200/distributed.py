"""Multi-GPU SGL transform: radial shells for the spherical stage, degree ranges
(l, all m) for the radial stage, one all-to-all in between (north star item 4).

The reference runs both stages of fsglft / ifsglft as thread-parallel loops in
one process -- over the 2B shells (sgl_transform.cpp:282-288) and over the B^2
(m, l) pairs (:294-308) -- with the `shells[i][nu]` buffer as the transpose
point.  Here every rank (one process per GPU, torch.distributed over NCCL):

forward
  1. spherical stage on its 2B/W shells -> S_local[nu][f][i_local] (all nu)
  2. all_to_all: the nu rows of degree range q go to rank q.  What rank q
     receives -- one block per source rank, S_r[nu - nu0_q][f][i_local] -- is
     exactly the shell-block layout the radial kernel reads in place, so there is
     no re-interleaving pass
  3. radial stage for its degrees -> its coefficients (disjoint omega entries)
  4. all_reduce(sum) assembles the omega-order vector on every rank (entries are
     disjoint, so the sum is exact)
inverse
  1. radial inverse for its degrees, written as one block per destination rank
  2. all_to_all back: rank r receives [nu][f][i_local] for its shells
  3. spherical inverse on its shells -> its psi-order slice of the samples

Degree ranges are balanced by the radial work (2l+1)(B-l) per degree.
Batched transforms need none of this: shard whole functions across ranks.

The compute is pluggable (`backend`): `CudaStages` drives the sm_100a kernels
through the C ABI (the product); the CPU test-suite drives the same
orchestration with a numpy model of the stages over gloo.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Partition:
    B: int
    world: int
    shells_per_rank: int
    l_ranges: list  # [(l0, l1)] per rank

    @staticmethod
    def make(B: int, world: int) -> "Partition":
        if (2 * B) % world != 0:
            raise ValueError(f"2B = {2 * B} shells do not split evenly over {world} ranks")
        work = np.array([(2 * l + 1) * (B - l) for l in range(B)], dtype=np.float64)
        cum = np.concatenate([[0.0], np.cumsum(work)])
        total = cum[-1]
        bounds = [0]
        for r in range(1, world):
            target = total * r / world
            l = int(np.searchsorted(cum, target))
            l = max(bounds[-1], min(B, l))
            bounds.append(l)
        bounds.append(B)
        return Partition(B, world, 2 * B // world, [(bounds[r], bounds[r + 1]) for r in range(world)])

    def nu_range(self, r: int):
        l0, l1 = self.l_ranges[r]
        return l0 * l0, l1 * l1

    def shell_range(self, r: int):
        return r * self.shells_per_rank, (r + 1) * self.shells_per_rank


class CudaStages:
    """Stage kernels through the C ABI on torch CUDA tensors (complex128)."""

    def __init__(self, plan):
        import paper_1604_05140_b200 as sgl

        self.sgl = sgl
        self.plan = plan
        self.L = sgl.lib()

    def _stream(self, t):
        import torch

        return torch.cuda.current_stream(t.device).cuda_stream

    def spherical_forward(self, samples_local, shell_begin, shell_count, batch):
        import torch

        B = self.plan.bandlimit
        out = torch.empty(B * B * batch * shell_count, dtype=torch.complex128, device=samples_local.device)
        self.sgl._check(self.L.sglgpu_spherical_forward(
            self.plan.handle, samples_local.data_ptr(), 4 * B * B * shell_count, out.data_ptr(), shell_begin,
            shell_count, batch, self._stream(out)))
        return out

    def radial_forward(self, blocks, l0, l1, shells_per_block, batch, coeffs_out):
        self.sgl._check(self.L.sglgpu_radial_forward(
            self.plan.handle, blocks.data_ptr(), coeffs_out.data_ptr(), l0, l1, shells_per_block, batch,
            self._stream(coeffs_out)))

    def radial_inverse(self, coeffs, l0, l1, shells_per_block, batch):
        import torch

        B = self.plan.bandlimit
        out = torch.empty((l1 * l1 - l0 * l0) * batch * 2 * B, dtype=torch.complex128, device=coeffs.device)
        self.sgl._check(self.L.sglgpu_radial_inverse(
            self.plan.handle, coeffs.data_ptr(), out.data_ptr(), l0, l1, shells_per_block, batch,
            self._stream(out)))
        return out

    def spherical_inverse(self, shells_local, shell_begin, shell_count, batch):
        import torch

        B = self.plan.bandlimit
        out = torch.empty(batch * 4 * B * B * shell_count, dtype=torch.complex128, device=shells_local.device)
        self.sgl._check(self.L.sglgpu_spherical_inverse(
            self.plan.handle, shells_local.data_ptr(), out.data_ptr(), 4 * B * B * shell_count, shell_begin,
            shell_count, batch, self._stream(out)))
        return out


def _a2a(dist, group, send, send_counts, recv_counts):
    """all_to_all_single on complex data (as float64 pairs, which gloo and NCCL both move)."""
    import torch

    recv = torch.empty(sum(recv_counts), dtype=torch.complex128, device=send.device)
    dist.all_to_all_single(torch.view_as_real(recv).reshape(-1), torch.view_as_real(send).reshape(-1),
                           output_split_sizes=[2 * c for c in recv_counts],
                           input_split_sizes=[2 * c for c in send_counts], group=group)
    return recv


def fsglft_distributed(samples_local, part: Partition, backend, dist, group=None, batch: int = 1):
    """Forward transform of `batch` functions whose psi-order shell slices
    [shell_begin, shell_end) of this rank are in `samples_local`
    ([batch, shells_per_rank * 4B^2] complex).  Returns the full omega-order
    coefficients [batch, Omega] on every rank."""
    import torch

    r = dist.get_rank(group)
    B, W, sc = part.B, part.world, part.shells_per_rank
    s0, _ = part.shell_range(r)
    S_local = backend.spherical_forward(samples_local, s0, sc, batch)       # [nu][f][i_local]
    row = batch * sc
    send_counts = [(part.nu_range(q)[1] - part.nu_range(q)[0]) * row for q in range(W)]
    nu0, nu1 = part.nu_range(r)
    recv_counts = [(nu1 - nu0) * row] * W
    blocks = _a2a(dist, group, S_local, send_counts, recv_counts)           # [src][nu - nu0][f][i_local]
    omega = B * (B + 1) * (2 * B + 1) // 6
    coeffs = torch.zeros((batch, omega), dtype=torch.complex128, device=samples_local.device)
    l0, l1 = part.l_ranges[r]
    if l1 > l0:
        backend.radial_forward(blocks, l0, l1, sc, batch, coeffs)
    dist.all_reduce(torch.view_as_real(coeffs), group=group)
    return coeffs


def ifsglft_distributed(coeffs, part: Partition, backend, dist, group=None, batch: int = 1):
    """Inverse transform: full coefficients [batch, Omega] (on every rank) ->
    this rank's psi-order shell slice [batch, shells_per_rank * 4B^2]."""
    r = dist.get_rank(group)
    B, W, sc = part.B, part.world, part.shells_per_rank
    l0, l1 = part.l_ranges[r]
    nu0, nu1 = part.nu_range(r)
    row = batch * sc
    if l1 > l0:
        blocks = backend.radial_inverse(coeffs, l0, l1, sc, batch)          # [dst][nu - nu0][f][i_local]
    else:
        import torch

        blocks = torch.empty(0, dtype=torch.complex128, device=coeffs.device)
    send_counts = [(nu1 - nu0) * row] * W
    recv_counts = [(part.nu_range(q)[1] - part.nu_range(q)[0]) * row for q in range(W)]
    S_local = _a2a(dist, group, blocks, send_counts, recv_counts)           # [nu][f][i_local]
    s0, _ = part.shell_range(r)
    return backend.spherical_inverse(S_local, s0, sc, batch)
