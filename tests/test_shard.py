"""Multi-rank partition of the λ launch on CPU (gloo, world_size 2 and 3): contiguous
ordinal chunks + static halo lists + all_to_all exchange reproduce the single-domain
CA exactly. Each rank updates only the tiles it owns (a numpy stepper standing in for
the device kernel), from a replica whose non-owned cells are stale except for the
exchanged halo cells — so a missing halo cell shows up as a wrong state."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from _oracle import orc_ca, orc_random_member_grid
from paper_2004_13475_b200.shard import ShardPlan, lambda_blocks, lambda_inverse_blocks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ca_owned_tiles(src: np.ndarray, plan: ShardPlan, birth=8, survive=12) -> np.ndarray:
    """One B/S step for the cells of this rank's tiles (others copied unchanged)."""
    n = src.shape[0]
    rho = plan.rho
    alive = (src != 0).astype(np.int64)
    yy, xx = np.mgrid[0:n, 0:n]
    member = (xx & (n - 1 - yy)) == 0
    alive &= member
    pad = np.pad(alive, 1)
    live = sum(pad[1 + dy:1 + dy + n, 1 + dx:1 + dx + n]
               for dy in (-1, 0, 1) for dx in (-1, 0, 1) if (dx, dy) != (0, 0))
    rule = np.where(alive == 1, (survive >> live) & 1, (birth >> live) & 1)
    nxt = (rule & member).astype(np.int64)
    out = src.copy()
    bx, by = plan.owned_blocks()
    for x0, y0 in zip(bx * rho, by * rho):
        out[y0:y0 + rho, x0:x0 + rho] = nxt[y0:y0 + rho, x0:x0 + rho]
    return out


def _worker(rank, world, port, r, rho, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = ShardPlan(r=r, rho=rho, world=world, rank=rank)
    g = torch.from_numpy(orc_random_member_grid(r, 1234, 2))
    # make non-owned cells stale garbage: only owned tiles + halos may be trusted
    own = np.zeros(g.shape, dtype=bool)
    t = np.arange(plan.begin, plan.begin + plan.count, dtype=np.int64)
    bx, by = lambda_blocks(t, plan.W)
    for x0, y0 in zip(bx * rho, by * rho):
        own[y0:y0 + rho, x0:x0 + rho] = True
    g[torch.from_numpy(~own)] = 7
    gather = lambda flat, idx: flat[idx].clone()  # noqa: E731
    def scatter(flat, idx, vals):
        flat[idx] = vals
    for _ in range(steps):
        plan.exchange_halo(g, dist, gather=gather, scatter=scatter)
        g = torch.from_numpy(_ca_owned_tiles(g.numpy(), plan))
    # collect owned tiles on rank 0
    full = torch.where(torch.from_numpy(own), g, torch.zeros_like(g))
    dist.all_reduce(full)
    if rank == 0:
        q.put((full.numpy(), plan.halo_cells_received()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,r,rho", [(2, 7, 8), (3, 7, 4), (2, 8, 16)])
def test_sharded_ca_matches_single_domain(world, r, rho):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(i, world, port, r, rho, 5, q)) for i in range(world)]
    for p in procs:
        p.start()
    got, halo = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = orc_ca(r, orc_random_member_grid(r, 1234, 2), 5)
    assert np.array_equal(got, want)
    assert halo > 0


def _compact_worker(rank, world, port, r, steps, q):
    """The compact-state partition: each rank holds a replica of the λ-ordered compact
    array, owns a contiguous range of the compact tile order, and exchanges halo cells by
    compact offset."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = ShardPlan(r=r, rho=32, world=world, rank=rank, state="compact")
    n = 1 << r
    cx, cy = lambda_blocks(np.arange(3 ** r, dtype=np.int64), 3 ** ((r + 1) // 2))  # λ of each slot
    tile = plan.tile_of_ordinal(lambda_inverse_blocks(cx >> 5, cy >> 5, plan.r_b, plan.W))
    own = torch.from_numpy(plan.owner(tile) == rank)
    g = torch.from_numpy(orc_random_member_grid(r, 1234, 2)[cy, cx].copy())
    g[~own] = 7  # stale garbage outside the owned slab
    gather = lambda flat, idx: flat[idx].clone()  # noqa: E731
    def scatter(flat, idx, vals):
        flat[idx] = vals
    for _ in range(steps):
        plan.exchange_halo(g, dist, gather=gather, scatter=scatter)
        emb = np.zeros((n, n), dtype=np.int64)
        emb[cy, cx] = g.numpy()
        nxt = _ca_owned_tiles(emb, plan)
        g = torch.where(own, torch.from_numpy(nxt[cy, cx].copy()), g)
    full = torch.where(own, g, torch.zeros_like(g))
    dist.all_reduce(full)
    if rank == 0:
        q.put((full.numpy(), plan.halo_cells_received()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,r", [(2, 7), (2, 10), (3, 10)])
def test_sharded_compact_ca_matches_single_domain(world, r):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_compact_worker, args=(i, world, port, r, 4, q)) for i in range(world)]
    for p in procs:
        p.start()
    got, halo = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cx, cy = lambda_blocks(np.arange(3 ** r, dtype=np.int64), 3 ** ((r + 1) // 2))
    want = orc_ca(r, orc_random_member_grid(r, 1234, 2), 4)[cy, cx]
    assert np.array_equal(got, want)
    assert halo > 0


def test_halo_lists_are_symmetric_and_small():
    """App. A.5: each tile needs <= 8 remote cells; what rank a receives from b is
    exactly what b sends to a."""
    r, rho = 12, 32
    for world, state in ((2, "embedded"), (4, "embedded"), (8, "embedded"), (2, "compact"), (8, "compact")):
        plans = [ShardPlan(r=r, rho=rho, world=world, rank=k, state=state) for k in range(world)]
        for a in range(world):
            assert sum(p.count for p in plans) == 3 ** (r - 5)
            for b in range(world):
                recv_ab = plans[a].recv_idx[sum(plans[a].recv_counts[:b]):
                                            sum(plans[a].recv_counts[:b + 1])]
                send_ba = plans[b].send_idx[sum(plans[b].send_counts[:a]):
                                            sum(plans[b].send_counts[:a + 1])]
                assert np.array_equal(recv_ab, send_ba)
            assert plans[a].halo_cells_received() <= 8 * plans[a].count


def test_lambda_inverse_blocks_round_trip():
    for r_b in range(0, 9):
        W = 3 ** ((r_b + 1) // 2)
        t = np.arange(3 ** r_b, dtype=np.int64)
        bx, by = lambda_blocks(t, W)
        assert np.array_equal(lambda_inverse_blocks(bx, by, r_b, W), t)


@pytest.mark.parametrize("r", [8, 10, 11])
def test_compact_segments_partition_the_state(r):
    """The compact RD / SW shard decomposition: each rank's (offset, count) runs are exactly the
    cells of its tiles (tile u = 9 compact rows x 27 columns at (9·u // H_b, 27·u % H_b)), and
    over the ranks they cover the 3^r values once."""
    W = 3 ** ((r + 1) // 2)
    for world in (1, 2, 3, 5, 8):
        cover = np.zeros(3 ** r, dtype=np.int64)
        for k in range(world):
            plan = ShardPlan(r=r, rho=32, world=world, rank=k, state="compact")
            segs = plan.compact_segments()
            assert len(segs) <= 19
            mine = np.concatenate([np.arange(o, o + c) for o, c in segs]) if segs else np.zeros(0, int)
            u = np.arange(plan.begin, plan.begin + plan.count)
            rows = (9 * (u // plan.Hb))[:, None] + np.arange(9)[None, :]
            want = (rows[:, :, None] * W + (27 * (u % plan.Hb))[:, None, None] +
                    np.arange(27)[None, None, :]).ravel()
            assert np.array_equal(np.sort(mine), np.sort(want)), (world, k)
            cover[mine] += 1
        assert np.all(cover == 1), world


def test_more_ranks_than_tiles_and_owner_table():
    """Empty shards (world > tiles) launch nothing and own nothing; the P2P owner table names,
    for every member halo cell of every tile, the rank whose tile range holds that cell."""
    for r, world in ((5, 3), (6, 5)):
        plans = [ShardPlan(r=r, rho=32, world=world, rank=k, state="compact") for k in range(world)]
        assert sum(p.count for p in plans) == 3 ** (r - 5)
        for p in plans:
            if p.count == 0:
                assert p.compact_segments() == []
    r, world = 10, 3
    plan = ShardPlan(r=r, rho=32, world=world, rank=1, state="compact")
    own = plan.halo_owner_table().reshape(-1, 8)
    n = 1 << r
    t = np.arange(plan.total, dtype=np.int64)
    bx, by = lambda_blocks(plan.ordinal_of_tile(t), plan.W)
    offs = np.array([(-1, -1), (0, -1), (1, -1), (-1, 31), (32, 30), (32, 31), (32, 32), (0, 32)])
    for k, (dx, dy) in enumerate(offs):
        cx, cy = bx * 32 + dx, by * 32 + dy
        ok = (cx >= 0) & (cy >= 0) & (cx < n) & (cy < n)
        ok &= (np.where(ok, cx, 0) & (n - 1 - np.where(ok, cy, 0))) == 0
        where = {(int(x), int(y)): int(u) for u, x, y in zip(t, bx, by)}  # tile at each λ block
        tile = np.array([where[(int(x) // 32, int(y) // 32)] for x, y in zip(cx[ok], cy[ok])], dtype=np.int64)
        assert np.array_equal(own[ok, k], plan.owner(tile)), k
        assert np.all(own[~ok, k] == 0)
