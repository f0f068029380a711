"""Slab decomposition host logic: topology, partition, coarse extents (CPU),
and the torch.distributed slab fabric with world_size 2 on gloo (CPU)."""

import os
import socket

import numpy as np
import pytest

from paper_2308_06085_b200.grid import BlockExtent, make_grid
from paper_2308_06085_b200.partition import (PartitionError, Topology, derive_coarse_extent,
                                             partition_grid, slab_partition, split_1d)


class TestTopology:
    def test_rank_order_example(self):        # reference Fig. "MPI topology" 3x4x5
        topo = Topology(3, 4, 5)
        assert topo.rank_of(1, 2, 0) == 7
        assert topo.coords_of(7) == (1, 2, 0)

    def test_round_trip_and_neighbors(self):
        topo = Topology(2, 2, 2)
        for r in range(topo.np):
            assert topo.rank_of(*topo.coords_of(r)) == r
        assert topo.neighbor(0, (0, -1)) is None
        assert topo.neighbor(0, (0, +1)) == 1 and topo.neighbor(0, (2, +1)) == 4

    def test_out_of_range(self):
        with pytest.raises(PartitionError):
            Topology(2, 2, 2).coords_of(8)


class TestPartition:
    def test_65_two_way(self):                # reference test_partition.py: 33 + 32
        ext = partition_grid(make_grid(65, 65, 65, 1 / 64), Topology(2))
        assert (ext[0].lo1, ext[0].hi1, ext[1].lo1, ext[1].hi1) == (1, 32, 33, 65)

    @pytest.mark.parametrize("n,p", [(33, 2), (65, 4), (129, 8), (17, 3), (9, 5)])
    def test_slabs_tile(self, n, p):
        grid = make_grid(n, n, n, 1.0 / (n - 1))
        cover = np.zeros(n, dtype=int)
        for e in slab_partition(grid, p):
            assert e.is_slab_of(grid)
            cover[e.lo1 - 1:e.hi1] += 1
        assert np.all(cover == 1)
        sizes = [e.nx for e in slab_partition(grid, p)]
        assert max(sizes) - min(sizes) <= 1

    def test_too_many_workers(self):
        with pytest.raises(PartitionError):
            split_1d(3, 4)

    def test_coarse_extent_alignment(self):   # reference: 33..65 -> 17..33
        f = partition_grid(make_grid(65, 65, 65, 1 / 64), Topology(2))
        c0, c1 = derive_coarse_extent(f[0]), derive_coarse_extent(f[1])
        assert (c0.lo1, c0.hi1, c1.lo1, c1.hi1) == (1, 16, 17, 33)

    @pytest.mark.parametrize("lo,width", [(1, 0), (2, 3), (7, 10), (33, 31), (4, 1)])
    def test_image_containment(self, lo, width):
        hi = lo + width
        c = derive_coarse_extent(BlockExtent(lo, lo, lo, hi, hi, hi))
        members = [i for i in range(1, hi + 2) if lo <= 2 * i - 1 <= hi]
        if members:
            assert (c.lo1, c.hi1) == (members[0], members[-1])
        else:
            assert c.is_empty()

    def test_native_coarse_slabs_match(self):
        """The native hierarchy derives the same coarse slabs (0-based rule)."""
        for lo0, nx in [(0, 33), (32, 33), (16, 17), (5, 11)]:
            clo, chi = (lo0 + 1) // 2, (lo0 + nx - 1) // 2
            c = derive_coarse_extent(BlockExtent(lo0 + 1, 1, 1, lo0 + nx, 9, 9))
            assert (c.lo1 - 1, c.hi1 - 1) == (clo, chi)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_2308_06085_b200._native import HF_GHOST
    from paper_2308_06085_b200.partition import TorchSlabComm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grid = make_grid(9, 5, 5, 0.25)
        e = slab_partition(grid, world)[rank]
        comm = TorchSlabComm()
        data = torch.zeros((e.nx + 2 * HF_GHOST, 5, 5), dtype=torch.complex128)
        i1 = torch.arange(e.lo1, e.hi1 + 1, dtype=torch.float64)
        data[HF_GHOST:HF_GHOST + e.nx] = (i1[:, None, None] + 1j * rank).expand(e.nx, 5, 5)
        comm.exchange([data], planes=2)
        total = comm.allreduce([complex(rank + 1, -rank)])
        part = torch.tensor([complex(rank + 1, -rank), complex(2 * rank, 1.0)], dtype=torch.complex128)
        dev_total = comm.allreduce_device([part]).numpy().copy()   # the device-resident driver's sums
        coarse = comm.allgather_planes(data[HF_GHOST:HF_GHOST + e.nx], [x.nx for x in slab_partition(grid, world)])
        out[rank] = (data.numpy().copy(), total, coarse.numpy().copy(), (e.lo1, e.hi1), dev_total)
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_halo_exchange():
    """world_size 2 on gloo: ghost planes hold the neighbour's boundary planes,
    the reduction is identical on both ranks, all-gather restores the field."""
    import torch.multiprocessing as mp
    from paper_2308_06085_b200._native import HF_GHOST
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    d0, t0, g0, (lo0, hi0), s0 = out[0]
    d1, t1, g1, (lo1, hi1), s1 = out[1]
    G = HF_GHOST
    nx0 = hi0 - lo0 + 1
    # rank 0's upper ghosts = rank 1's first two planes (global planes lo1, lo1+1)
    assert np.all(d0[G + nx0] == lo1 + 1j) and np.all(d0[G + nx0 + 1] == lo1 + 1 + 1j)
    # rank 1's lower ghosts = rank 0's last two planes
    assert np.all(d1[G - 1] == hi0) and np.all(d1[G - 2] == hi0 - 1)
    # physical faces untouched
    assert np.all(d0[:G] == 0) and np.all(d1[G + (hi1 - lo1 + 1):] == 0)
    assert t0 == t1 == complex(3, -1)
    np.testing.assert_array_equal(s0, s1)
    np.testing.assert_array_equal(s0, np.array([3 - 1j, 2 + 2j]))
    np.testing.assert_array_equal(g0, g1)
    assert g0.shape[0] == 9 and np.all(g0[:, 0, 0].real == np.arange(1, 10))
