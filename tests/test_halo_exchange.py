"""Host logic of the multi-process compact CA over NCCL (nbb_gpu_ca_compact_comm_dev): the halo
exchange lists (nbb_gpu_halo_exchange_counts / _lists, nbbhost::halo_exchange_lists).

Each rank owns the contiguous chunk of compact tiles of shard.compact_shard_chunk (ceil(tiles / world) rounded up to whole cluster columns; dispatch.cpp:419-427).
Before a pass of K steps it must hold every cell of another rank that can reach one of its
members within K steps. Checked here without a GPU:
  * K = 1 equals the one-step exchange of the Python shard plan (shard.ShardPlan, state="compact"),
    which the gloo / NCCL exchange tests already pin to the single-GPU step;
  * for K up to 8 the lists contain every cell a breadth-first search over member cells finds
    within K steps of the rank's tiles (brute force on the embedded grid), lie in the sender's
    tiles, are symmetric (rank i's send to j == rank j's receive from i) and grow with K."""
import ctypes

import numpy as np
import pytest

from paper_2004_13475_b200 import _abi, shard
from paper_2004_13475_b200.nbb import DispatchConfig


def lists(r, world, rank, kmax):
    lib = _abi.load()
    c = DispatchConfig(r=r, rho=32).to_c()
    sc = (ctypes.c_uint64 * world)()
    rc = (ctypes.c_uint64 * world)()
    assert lib.nbb_gpu_halo_exchange_counts(ctypes.byref(c), world, rank, kmax, sc, rc) == 0, \
        lib.nbb_gpu_last_error()
    send, recv = [], []
    for p in range(world):
        s = np.zeros(max(1, sc[p]), dtype=np.uint32)
        v = np.zeros(max(1, rc[p]), dtype=np.uint32)
        assert lib.nbb_gpu_halo_exchange_lists(ctypes.byref(c), world, rank, kmax, p,
                                               s.ctypes.data_as(ctypes.c_void_p),
                                               v.ctypes.data_as(ctypes.c_void_p)) == 0
        send.append(s[:sc[p]].astype(np.int64))
        recv.append(v[:rc[p]].astype(np.int64))
    return send, recv


def tile_of_offset(off, r):
    """The compact tile u = ωx_b·H_b + ωy_b holding compact offset `off`."""
    W, Hb = 3 ** ((r + 1) // 2), 3 ** ((r - 5) // 2)
    row, col = off // W, off % W
    return (row // 9) * Hb + col // 27


@pytest.mark.parametrize("r,world", [(6, 2), (8, 3), (10, 2), (10, 4), (11, 5)])
def test_one_step_lists_equal_shard_plan(r, world):
    for rank in range(world):
        send, recv = lists(r, world, rank, 1)
        plan = shard.ShardPlan(r=r, rho=32, world=world, rank=rank, state="compact")
        so = np.cumsum([0] + plan.send_counts)
        ro = np.cumsum([0] + plan.recv_counts)
        for p in range(world):
            assert np.array_equal(np.sort(plan.recv_idx[ro[p]:ro[p + 1]]), recv[p]), (rank, p)
            assert np.array_equal(np.sort(plan.send_idx[so[p]:so[p + 1]]), send[p]), (rank, p)


@pytest.mark.parametrize("r,world", [(7, 2), (11, 3), (10, 8), (12, 4)])
def test_lists_symmetric_and_owned(r, world):
    W, Hb = 3 ** ((r + 1) // 2), 3 ** ((r - 5) // 2)
    tiles = 3 ** (r - 5)
    chunk = shard.compact_shard_chunk(r - 5, tiles, Hb, world)
    for k in (2, 5, 8):
        al = [lists(r, world, q, k) for q in range(world)]
        for i in range(world):
            for j in range(world):
                assert np.array_equal(al[i][0][j], al[j][1][i]), (k, i, j)  # send i->j == recv j<-i
                if i != j and al[i][1][j].size:
                    assert np.all(tile_of_offset(al[i][1][j], r) // chunk == j)  # in the sender's tiles
            assert al[i][1][i].size == 0
        small = [lists(r, world, q, k - 1) for q in range(world)]
        for i in range(world):
            for j in range(world):
                assert np.isin(small[i][1][j], al[i][1][j]).all()  # grows with K


@pytest.mark.parametrize("r,world,k", [(7, 3, 3), (10, 3, 3), (10, 2, 6), (11, 4, 8)])
def test_lists_cover_the_k_step_neighbourhood(r, world, k):
    """Brute force: BFS over member cells from every member of the rank's tiles, k layers; every
    reached cell owned by another rank is in the receive list from that rank."""
    n = 1 << r
    W = 3 ** ((r + 1) // 2)
    tiles = 3 ** (r - 5)
    chunk = shard.compact_shard_chunk(r - 5, tiles, 3 ** ((r - 5) // 2), world)
    ys, xs = np.nonzero(((np.arange(n)[None, :] & ~np.arange(n)[:, None]) == 0))  # x ⊆ y
    member = np.zeros((n, n), dtype=bool)
    member[ys, xs] = True
    comp = shard.lambda_inverse_blocks(xs, ys, r, W)  # compact offset ωy·W + ωx of each member
    offset = np.full((n, n), -1, dtype=np.int64)
    offset[ys, xs] = comp
    owner = np.full((n, n), -1, dtype=np.int64)
    owner[ys, xs] = tile_of_offset(comp, r) // chunk
    for rank in range(world):
        _, recv = lists(r, world, rank, k)
        frontier = (owner == rank)
        seen = frontier.copy()
        for _ in range(k):
            pad = np.pad(frontier, 1)
            grown = np.zeros_like(frontier)
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    if dx or dy:
                        grown |= pad[1 + dy:1 + dy + n, 1 + dx:1 + dx + n]
            grown &= member & ~seen
            seen |= grown
            frontier = grown
        reached = seen & (owner != rank) & (owner >= 0)
        for p in range(world):
            need = np.unique(offset[reached & (owner == p)])
            assert np.isin(need, recv[p]).all(), (rank, p, np.setdiff1d(need, recv[p])[:5])
