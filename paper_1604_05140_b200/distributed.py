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

The fused variant (`fsglft_distributed_fused` / `ifsglft_distributed_fused`)
replaces the all-to-all by NVLink peer stores from the producing kernel's
epilogue into the consumers' receive buffers (mapped with CUDA IPC,
`PeerBuffers`), so the exchange overlaps the Legendre / radial-inverse GEMM
tile by tile; a one-element all_reduce on the stream orders the stores.  The
coefficient assembly is fused the same way: each rank's radial-forward epilogue
stores its degrees into every rank's coefficient vectors (no all-reduce).

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


# ---------------------------------------------------------------- fused exchange over NVLink
class PeerBuffers:
    """Receive buffers of the fused exchange and every rank's view of them.

    fwd[q]: rank q's forward receive buffer, W shell blocks [src][nu - nu0_q][f][i_local]
            (what sglgpu_radial_forward reads in place);
    inv[b]: rank b's inverse buffer S[nu][f][i_local] over all nu (what
            sglgpu_spherical_inverse reads).
    On a node the peers' buffers are mapped with CUDA IPC (`exchange`); `local`
    builds the same structure for W virtual ranks on one device (tests)."""

    def __init__(self, part: "Partition", batch: int, fwd_ptrs, inv_ptrs, owned, opened, coef_ptrs=None):
        self.part, self.batch = part, batch
        self.fwd, self.inv = fwd_ptrs, inv_ptrs
        self.coef = coef_ptrs or []  # coef[q]: rank q's omega-order coefficient vectors (batch x Omega)
        self._owned, self._opened = owned, opened

    @staticmethod
    def sizes(part: "Partition", batch: int, q: int):
        row = batch * part.shells_per_rank  # complex per nu row of a shell block
        nu0, nu1 = part.nu_range(q)
        return part.world * (nu1 - nu0) * row * 16, part.B * part.B * row * 16

    @staticmethod
    def coef_bytes(part: "Partition", batch: int):
        B = part.B
        return batch * (B * (B + 1) * (2 * B + 1) // 6) * 16

    @staticmethod
    def _alloc(L, nbytes):
        import ctypes

        import paper_1604_05140_b200 as sgl

        p = ctypes.c_void_p()
        sgl._check(L.sglgpu_device_alloc(nbytes, ctypes.byref(p)))
        return p.value

    @classmethod
    def local(cls, part: "Partition", batch: int):
        import paper_1604_05140_b200 as sgl

        L = sgl.lib()
        fwd, inv, coef = [], [], []
        for q in range(part.world):
            fb, ib = cls.sizes(part, batch, q)
            fwd.append(cls._alloc(L, fb))
            inv.append(cls._alloc(L, ib))
            coef.append(cls._alloc(L, cls.coef_bytes(part, batch)))
        return cls(part, batch, fwd, inv, fwd + inv + coef, [], coef)

    @classmethod
    def exchange(cls, part: "Partition", batch: int, dist, group=None):
        """Allocates this rank's buffers, all-gathers their IPC handles and maps the peers'."""
        import ctypes

        import paper_1604_05140_b200 as sgl

        L = sgl.lib()
        r, W = dist.get_rank(group), part.world
        fb, ib = cls.sizes(part, batch, r)
        mine = [cls._alloc(L, fb), cls._alloc(L, ib), cls._alloc(L, cls.coef_bytes(part, batch))]
        handles = []
        for p in mine:
            h = ctypes.create_string_buffer(64)
            sgl._check(L.sglgpu_ipc_export(p, h))
            handles.append(h.raw)
        allh = [None] * W
        dist.all_gather_object(allh, handles, group=group)
        fwd, inv, coef, opened = [], [], [], []
        for q in range(W):
            if q == r:
                fwd.append(mine[0])
                inv.append(mine[1])
                coef.append(mine[2])
                continue
            ptrs = []
            for h in allh[q]:
                p = ctypes.c_void_p()
                sgl._check(L.sglgpu_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(p)))
                ptrs.append(p.value)
                opened.append(p.value)
            fwd.append(ptrs[0])
            inv.append(ptrs[1])
            coef.append(ptrs[2])
        return cls(part, batch, fwd, inv, mine, opened, coef)

    def close(self):
        import paper_1604_05140_b200 as sgl

        L = sgl.lib()
        for p in self._opened:
            L.sglgpu_ipc_close(p)
        for p in self._owned:
            L.sglgpu_device_free(p)
        self._opened, self._owned = [], []

    def fwd_dst(self, r: int):
        """Where rank r's shell block starts in every rank's forward receive buffer."""
        import ctypes

        part, row = self.part, self.batch * self.part.shells_per_rank
        out = []
        for q in range(part.world):
            nu0, nu1 = part.nu_range(q)
            out.append(self.fwd[q] + r * (nu1 - nu0) * row * 16)
        return (ctypes.c_void_p * part.world)(*out)

    def inv_dst(self):
        import ctypes

        return (ctypes.c_void_p * self.part.world)(*self.inv)

    def coef_dst(self):
        import ctypes

        return (ctypes.c_void_p * self.part.world)(*self.coef)

    def coef_tensor(self, r: int):
        """Rank r's coefficient vectors as a (batch, Omega) complex128 CUDA tensor view."""
        import torch

        B = self.part.B
        omega = B * (B + 1) * (2 * B + 1) // 6

        class _View:  # __cuda_array_interface__ over the raw allocation
            __cuda_array_interface__ = {"shape": (self.batch, omega), "typestr": "<c16",
                                        "data": (self.coef[r], False), "version": 3, "strides": None}

        return torch.as_tensor(_View(), device="cuda")


def _stream_of(t):
    import torch

    return torch.cuda.current_stream(t.device).cuda_stream


def fused_forward_spherical(samples_local, part: "Partition", stages: "CudaStages", peers: PeerBuffers, rank: int,
                            batch: int = 1):
    """Step 1 of the fused forward: rank `rank`'s spherical stage, its S rows stored
    straight into their owners' receive buffers (sglgpu_spherical_forward_to)."""
    import ctypes

    B, W, sc = part.B, part.world, part.shells_per_rank
    s0, _ = part.shell_range(rank)
    bounds = (ctypes.c_int * (W + 1))(*([lr[0] for lr in part.l_ranges] + [B]))
    stages.sgl._check(stages.L.sglgpu_spherical_forward_to(
        stages.plan.handle, samples_local.data_ptr(), 4 * B * B * sc, s0, sc, batch, W, peers.fwd_dst(rank), bounds,
        _stream_of(samples_local)))


def fused_forward_radial(part: "Partition", stages: "CudaStages", peers: PeerBuffers, rank: int, coeffs):
    """Step 2: the radial stage of rank `rank` on its receive buffer (in place) -> its
    degrees of `coeffs` ([batch, Omega], other entries untouched)."""
    l0, l1 = part.l_ranges[rank]
    if l1 > l0:
        stages.sgl._check(stages.L.sglgpu_radial_forward(
            stages.plan.handle, peers.fwd[rank], coeffs.data_ptr(), l0, l1, part.shells_per_rank, peers.batch,
            _stream_of(coeffs)))


def fused_forward_radial_bcast(part: "Partition", stages: "CudaStages", peers: PeerBuffers, rank: int, stream=None):
    """Step 2 with the assembly fused in: rank `rank`'s radial stage stores its
    degrees into EVERY rank's coefficient vectors (peers.coef, NVLink peer stores
    from the GEMM epilogue; sglgpu_radial_forward_to) -- no all-reduce."""
    l0, l1 = part.l_ranges[rank]
    if l1 > l0:
        stages.sgl._check(stages.L.sglgpu_radial_forward_to(
            stages.plan.handle, peers.fwd[rank], l0, l1, part.shells_per_rank, peers.batch, part.world,
            peers.coef_dst(), stream))


def fused_inverse_radial(coeffs, part: "Partition", stages: "CudaStages", peers: PeerBuffers, rank: int):
    """Step 1 of the fused inverse: rank `rank`'s radial stage, each shell block
    stored straight into the shell owner's S buffer (sglgpu_radial_inverse_to)."""
    l0, l1 = part.l_ranges[rank]
    if l1 > l0:
        stages.sgl._check(stages.L.sglgpu_radial_inverse_to(
            stages.plan.handle, coeffs.data_ptr(), l0, l1, part.shells_per_rank, peers.batch, part.world,
            peers.inv_dst(), _stream_of(coeffs)))


def fused_inverse_spherical(part: "Partition", stages: "CudaStages", peers: PeerBuffers, rank: int, device):
    """Step 2: the spherical inverse of rank `rank`'s shells from its S buffer."""
    import torch

    B, sc = part.B, part.shells_per_rank
    out = torch.empty(peers.batch * 4 * B * B * sc, dtype=torch.complex128, device=device)
    stages.sgl._check(stages.L.sglgpu_spherical_inverse(
        stages.plan.handle, peers.inv[rank], out.data_ptr(), 4 * B * B * sc, part.shell_range(rank)[0], sc,
        peers.batch, _stream_of(out)))
    return out


def _stream_barrier(dist, group, device):
    """Orders every rank's peer stores before any rank reads its receive buffer:
    a one-element all_reduce is stream-ordered on each rank (NCCL)."""
    import torch

    t = torch.zeros(1, device=device)
    dist.all_reduce(t, group=group)


def fsglft_distributed_fused(samples_local, part: "Partition", stages: "CudaStages", peers: PeerBuffers, dist,
                             group=None, batch: int = 1):
    """fsglft_distributed with the all-to-all fused into the Legendre epilogue
    (NVLink peer stores into the owners' receive buffers; see PeerBuffers)."""
    import torch

    if batch != peers.batch:  # the receive buffers and the peer offsets are sized for peers.batch
        raise ValueError(f"fsglft_distributed_fused: batch {batch} != the peer buffers' batch {peers.batch}")
    r = dist.get_rank(group)
    fused_forward_spherical(samples_local, part, stages, peers, r, batch)
    _stream_barrier(dist, group, samples_local.device)
    if peers.coef and part.world > 1:
        # every rank's radial stage stores its degrees into all ranks' vectors
        # (at one rank the all-reduce below is free and the extra barrier is not)
        fused_forward_radial_bcast(part, stages, peers, r, _stream_of(samples_local))
        _stream_barrier(dist, group, samples_local.device)
        return peers.coef_tensor(r).clone()
    omega = part.B * (part.B + 1) * (2 * part.B + 1) // 6
    coeffs = torch.zeros((batch, omega), dtype=torch.complex128, device=samples_local.device)
    fused_forward_radial(part, stages, peers, r, coeffs)
    dist.all_reduce(torch.view_as_real(coeffs), group=group)
    return coeffs


def ifsglft_distributed_fused(coeffs, part: "Partition", stages: "CudaStages", peers: PeerBuffers, dist,
                              group=None, batch: int = 1):
    """ifsglft_distributed with the all-to-all fused into the radial-inverse epilogue.

    Ends with a stream barrier: the next call's radial-inverse peer stores go
    into every rank's S buffer, which this call's spherical inverse on that rank
    may still be reading (the forward path is ordered by its own trailing
    collective)."""
    if batch != peers.batch:
        raise ValueError(f"ifsglft_distributed_fused: batch {batch} != the peer buffers' batch {peers.batch}")
    r = dist.get_rank(group)
    fused_inverse_radial(coeffs, part, stages, peers, r)
    _stream_barrier(dist, group, coeffs.device)
    out = fused_inverse_spherical(part, stages, peers, r, coeffs.device)
    _stream_barrier(dist, group, coeffs.device)
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
