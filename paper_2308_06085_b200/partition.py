"""Slab decomposition, halo exchange and inner-product reductions.

Mirrors /root/reference/pkg/src/helmfree/partition.py: Topology (:56-92),
_split_1d (:95-100), partition_grid (:103-117), derive_coarse_extent
(:120-131), Exchanger.exchange (:509-536), DistContext.dot / norm
(:611-621).  B200 layout: the grid is split into slabs along i1 only (one
process per GPU, npx0 = world size), so a halo is HF_GHOST contiguous planes
of n2*n3 complex values per face, sent peer-to-peer (NCCL over NVLink on
GPUs, gloo on CPU); NCCL all-reduce is used only for inner products.

Two fabrics share one interface:
  * TorchSlabComm  -- one slab per process, torch.distributed P2P + all_reduce;
  * LocalSlabComm  -- several slabs in one process (virtual ranks), halos by
                      tensor copies; used to run the multi-slab path on one GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._native import HF_GHOST
from .grid import BlockExtent, Grid3

__all__ = ["PartitionError", "Topology", "split_1d", "partition_grid", "derive_coarse_extent",
           "slab_partition", "TorchSlabComm", "LocalSlabComm"]


class PartitionError(ValueError):
    pass


@dataclass(frozen=True)
class Topology:
    """Cartesian worker layout, x-line lexicographic ranks (partition.py:56-92)."""

    npx0: int
    npy0: int = 1
    npz0: int = 1

    @property
    def np(self) -> int:
        return self.npx0 * self.npy0 * self.npz0

    @property
    def dims(self):
        return (self.npx0, self.npy0, self.npz0)

    def rank_of(self, npx, npy, npz) -> int:
        if not (0 <= npx < self.npx0 and 0 <= npy < self.npy0 and 0 <= npz < self.npz0):
            raise PartitionError(f"coords {(npx, npy, npz)} outside {self.dims}")
        return npx + npy * self.npx0 + npz * self.npx0 * self.npy0

    def coords_of(self, rank):
        if not 0 <= rank < self.np:
            raise PartitionError(f"rank {rank} outside 0..{self.np - 1}")
        return (rank % self.npx0, (rank // self.npx0) % self.npy0, rank // (self.npx0 * self.npy0))

    def neighbor(self, rank, face):
        dim, side = face
        c = list(self.coords_of(rank))
        c[dim] += side
        if not 0 <= c[dim] < self.dims[dim]:
            return None
        return self.rank_of(*c)


def split_1d(n: int, parts: int):
    """Balanced contiguous split of 1..n (partition.py:95-100)."""
    if parts > n:
        raise PartitionError(f"cannot split {n} vertices over {parts} workers")
    bounds = [(p * n) // parts for p in range(parts + 1)]
    return [(bounds[p] + 1, bounds[p + 1]) for p in range(parts)]


def partition_grid(grid: Grid3, topo: Topology):
    """Blockwise partition, one extent per rank (partition.py:103-117)."""
    sx, sy, sz = split_1d(grid.n1, topo.npx0), split_1d(grid.n2, topo.npy0), split_1d(grid.n3, topo.npz0)
    out = []
    for rank in range(topo.np):
        px, py, pz = topo.coords_of(rank)
        out.append(BlockExtent(sx[px][0], sy[py][0], sz[pz][0], sx[px][1], sy[py][1], sz[pz][1]))
    return out


def derive_coarse_extent(fine: BlockExtent) -> BlockExtent:
    """Coarse vertices whose fine image 2i-1 lies in the block (partition.py:120-131)."""
    clo = tuple((lo + 2) // 2 for lo in fine.lo)
    chi = tuple((hi + 1) // 2 for hi in fine.hi)
    return BlockExtent(clo[0], clo[1], clo[2], chi[0], chi[1], chi[2])


def slab_partition(grid: Grid3, nslabs: int):
    """The B200 decomposition: npx0 = nslabs slabs along i1."""
    return partition_grid(grid, Topology(nslabs, 1, 1))


class _SlabCommBase:
    """Halo planes of a device field laid out as (nx + 2G, n2, n3)."""

    @staticmethod
    def _planes(data, nx, which, planes):
        G = HF_GHOST
        if which == "send_lo":
            return data[G:G + planes]
        if which == "send_hi":
            return data[G + nx - planes:G + nx]
        if which == "recv_lo":
            return data[G - planes:G]
        return data[G + nx:G + nx + planes]


class TorchSlabComm(_SlabCommBase):
    """One slab per process over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    @property
    def local_ranks(self):
        return [self.rank]

    def exchange(self, fields, planes: int = 1):
        """fields: [data tensor] of this rank's slab; fills `planes` ghost planes per face."""
        dist = self.dist
        (data,) = fields
        nx = data.shape[0] - 2 * HF_GHOST
        ops = []
        lo = self.rank - 1 if self.rank > 0 else None
        hi = self.rank + 1 if self.rank < self.size - 1 else None
        if lo is not None:
            ops.append(dist.P2POp(dist.isend, self._planes(data, nx, "send_lo", planes), lo, self.group))
            ops.append(dist.P2POp(dist.irecv, self._planes(data, nx, "recv_lo", planes), lo, self.group))
        if hi is not None:
            ops.append(dist.P2POp(dist.isend, self._planes(data, nx, "send_hi", planes), hi, self.group))
            ops.append(dist.P2POp(dist.irecv, self._planes(data, nx, "recv_hi", planes), hi, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def allreduce(self, values):
        """values: [complex] of this rank -> global sum (same on every rank)."""
        import torch
        t = torch.tensor([values[0].real, values[0].imag], dtype=torch.float64)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, group=self.group)
        t = t.cpu()
        return complex(float(t[0]), float(t[1]))

    def allreduce_device(self, tensors):
        """tensors: [device tensor of partial sums] of this rank -> the global sum
        as a device tensor, without a host round trip on NCCL (one all-reduce)."""
        (t,) = tensors
        if self.dist.get_backend(self.group) == "nccl":
            out = t.clone()
            self.dist.all_reduce(self._real(out), group=self.group)
            return out
        host = t.cpu()                      # gloo: host tensors
        self.dist.all_reduce(self._real(host), group=self.group)
        return host.to(t.device)

    @staticmethod
    def _real(t):
        import torch
        return torch.view_as_real(t) if t.is_complex() else t

    def allgather_planes(self, owned, counts):
        """Concatenate every rank's owned planes (coarsest level) in rank order."""
        import torch
        cmax = max(counts)                 # all_gather needs equal sizes: pad to the largest slab
        tail = tuple(owned.shape[1:])
        mine = torch.zeros((cmax,) + tail, dtype=owned.dtype, device=owned.device)
        mine[:owned.shape[0]] = owned
        parts = [torch.empty((cmax,) + tail, dtype=owned.dtype, device=owned.device) for _ in counts]
        self.dist.all_gather(parts, mine, group=self.group)
        return torch.cat([p[:c] for p, c in zip(parts, counts)], 0)


class LocalSlabComm(_SlabCommBase):
    """All slabs of the decomposition in this process (virtual ranks)."""

    def __init__(self, nslabs: int):
        self.size = nslabs
        self.rank = 0

    @property
    def local_ranks(self):
        return list(range(self.size))

    def exchange(self, fields, planes: int = 1):
        nxs = [d.shape[0] - 2 * HF_GHOST for d in fields]
        for r in range(self.size - 1):
            a, b = fields[r], fields[r + 1]
            self._planes(a, nxs[r], "recv_hi", planes).copy_(self._planes(b, nxs[r + 1], "send_lo", planes))
            self._planes(b, nxs[r + 1], "recv_lo", planes).copy_(self._planes(a, nxs[r], "send_hi", planes))

    def allreduce(self, values):
        tot = 0j
        for v in values:           # fixed rank order
            tot += v
        return tot

    def allreduce_device(self, tensors):
        """Per-slab partial sums -> their total (fixed slab order, on the device)."""
        tot = tensors[0].clone()
        for t in tensors[1:]:
            tot += t
        return tot

    def allgather_planes(self, owned_list, counts):
        import torch
        return torch.cat(list(owned_list), 0)
