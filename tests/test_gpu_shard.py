"""The multi-GPU CA path on one B200: world_size ranks (gloo, all on cuda:0) each
launch only their contiguous chunk of λ tiles (nbb_config.shard_begin/count) on a
full replica, exchange the halo cells with the library's gather/scatter kernels
before every step, and together reproduce the single-domain oracle exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from _oracle import orc_ca, orc_random_member_grid

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, r, rho, steps, cell_width, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2004_13475_b200 import device as dev
    from paper_2004_13475_b200 import nbb
    from paper_2004_13475_b200.shard import ShardPlan, lambda_blocks, lambda_inverse_blocks
    n = 1 << r
    compact = cell_width == "compact"
    plan = ShardPlan(r=r, rho=rho, world=world, rank=rank, state="compact" if compact else "embedded")
    g = orc_random_member_grid(r, 4321, 2)
    if compact:  # the λ-ordered compact state: slot c holds cell λ(c)
        cx, cy = lambda_blocks(np.arange(3 ** r, dtype=np.int64), 3 ** ((r + 1) // 2))
        a = torch.from_numpy(g[cy, cx].copy()).cuda()
        c = nbb.DispatchConfig(r=r, rho=rho, max_cells=n * n)
    else:
        dt = torch.int64 if cell_width == 8 else torch.uint8
        a = torch.from_numpy(g).to(dt).cuda()
        c = nbb.DispatchConfig(r=r, rho=rho, max_cells=n * n, cell_width=cell_width)
    b = torch.zeros_like(a)
    lc = plan.local_config(c)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(steps):
        plan.exchange_halo(a, dist)
        if compact:
            dev.ca_compact_step_dev(lc, a.data_ptr(), b.data_ptr(), nbb.CaRule(), s)
        else:
            dev.ca_step_dev(lc, a.data_ptr(), b.data_ptr(), nbb.CaRule(), s)
        a, b = b, a
    torch.cuda.synchronize()
    if compact:
        tile = plan.tile_of_ordinal(lambda_inverse_blocks(cx >> 5, cy >> 5, plan.r_b, plan.W))
        mine_c = torch.where(torch.from_numpy(plan.owner(tile) == rank), a.cpu(), torch.zeros_like(a.cpu()))
        mine = torch.zeros(n, n, dtype=torch.int64)
        mine[torch.from_numpy(cy), torch.from_numpy(cx)] = mine_c
    else:
        own = np.zeros((n, n), dtype=bool)
        bx, by = plan.owned_blocks()
        for x0, y0 in zip(bx * rho, by * rho):
            own[y0:y0 + rho, x0:x0 + rho] = True
        mine = torch.where(torch.from_numpy(own), a.cpu().to(torch.int64),
                           torch.zeros(n, n, dtype=torch.int64))
    dist.all_reduce(mine)
    if rank == 0:
        q.put(mine.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,r,rho,cw", [(2, 10, 32, 8), (3, 10, 16, 8), (2, 11, 32, 1),
                                           (2, 10, 32, "compact"), (3, 11, 32, "compact")])
def test_sharded_ca_on_gpu(world, r, rho, cw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    steps = 6
    procs = [ctx.Process(target=_worker, args=(i, world, port, r, rho, steps, cw, q)) for i in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = orc_ca(r, orc_random_member_grid(r, 4321, 2), steps)
    assert np.array_equal(got, want)


def _p2p_worker(rank, world, port, r, steps, q, mode="step", birth=8, survive=12):
    """The P2P compact CA: ranks on one B200 share buffers through CUDA IPC mappings."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2004_13475_b200 import nbb
    from paper_2004_13475_b200.shard import (P2PCompactCA, ShardPlan, lambda_blocks,
                                             lambda_inverse_blocks)
    n = 1 << r
    plan = ShardPlan(r=r, rho=32, world=world, rank=rank, state="compact")
    cx, cy = lambda_blocks(np.arange(3 ** r, dtype=np.int64), 3 ** ((r + 1) // 2))
    tile = plan.tile_of_ordinal(lambda_inverse_blocks(cx >> 5, cy >> 5, plan.r_b, plan.W))
    own = torch.from_numpy(plan.owner(tile) == rank)
    init = torch.from_numpy(orc_random_member_grid(r, 4321, 2)[cy, cx].copy())
    init[~own] = 7  # only this rank's tiles are trusted: remote cells must come from peers
    ca = P2PCompactCA(plan, dist, device=0, timeout_ms=60000, two_step=(mode == "passes"))
    ca.load(init)
    c = nbb.DispatchConfig(r=r, rho=32, max_cells=n * n)
    s = torch.cuda.current_stream().cuda_stream
    rule = nbb.CaRule(birth=birth, survive=survive)
    if mode == "step":  # one call per step
        for _ in range(steps):
            ca.step(c, rule, s)
    else:  # two calls: the pass parity and arrival targets carry across calls
        ca.run(c, rule, steps // 2 + 1, s)
        ca.run(c, rule, steps - steps // 2 - 1, s)
    ca.check(s)
    out = ca.state().cpu()
    mine_c = torch.where(own, out, torch.zeros_like(out))
    mine = torch.zeros(n, n, dtype=torch.int64)
    mine[torch.from_numpy(cy), torch.from_numpy(cx)] = mine_c
    ca.close()
    dist.all_reduce(mine)
    if rank == 0:
        q.put(mine.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,r,mode,steps,rule", [
    (2, 10, "step", 6, (8, 12)), (3, 11, "step", 6, (8, 12)), (4, 12, "step", 6, (8, 12)),
    # passes of two steps (ca_compact2_kernel over peer memory), odd and even step counts,
    # the B3/S23 and the generic-rule instantiations
    (2, 10, "passes", 7, (8, 12)), (3, 11, "passes", 6, (8, 12)), (4, 12, "passes", 9, (8, 12)),
    (3, 10, "passes", 8, (72, 12)), (2, 12, "single", 5, (8, 12))])
def test_p2p_compact_ca_on_gpu(world, r, mode, steps, rule):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(i, world, port, r, steps, q, mode, *rule))
             for i in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = orc_ca(r, orc_random_member_grid(r, 4321, 2), steps, *rule)
    assert np.array_equal(got, want)


def _rd_worker(rank, world, port, r, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2004_13475_b200 import nbb
    from paper_2004_13475_b200.shard import (ShardPlan, lambda_blocks, sharded_reduction,
                                             sharded_single_write)
    n = 1 << r
    # values near 2^62 so the int64 sum wraps, as the reference's accumulation does
    g = orc_random_member_grid(r, 99, 1 << 62)
    c = nbb.DispatchConfig(r=r, rho=32, max_cells=n * n)
    out = {}
    for state in ("embedded", "compact"):
        plan = ShardPlan(r=r, rho=32, world=world, rank=rank, state=state)
        if state == "compact":
            cx, cy = lambda_blocks(np.arange(3 ** r, dtype=np.int64), 3 ** ((r + 1) // 2))
            a = torch.from_numpy(g[cy, cx].copy()).cuda()
        else:
            a = torch.from_numpy(g.copy()).cuda()
        out[state] = sharded_reduction(plan, c, a.data_ptr(), dist,
                                       torch.cuda.current_stream().cuda_stream)
        b = torch.zeros_like(a)
        sharded_single_write(plan, c, b.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        bh = b.cpu()
        dist.all_reduce(bh)  # every rank wrote only its own tiles: the sum is the full write
        out[state + "_sw"] = bh.numpy()
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,r", [(2, 10), (3, 11)])
def test_sharded_reduction_and_single_write(world, r):
    """RD = per-rank partial sums over each rank's tiles + ONE all-reduce; SW = each rank writes
    its own tiles. Both states, values that make the int64 sum wrap."""
    from _oracle import orc_reduction, orc_single_write
    from paper_2004_13475_b200.shard import lambda_blocks
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rd_worker, args=(i, world, port, r, q)) for i in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = orc_random_member_grid(r, 99, 1 << 62)
    want = orc_reduction(r, g)
    assert got["embedded"] == want and got["compact"] == want
    sw = orc_single_write(r)
    assert np.array_equal(got["embedded_sw"], sw)
    cx, cy = lambda_blocks(np.arange(3 ** r, dtype=np.int64), 3 ** ((r + 1) // 2))
    assert np.array_equal(got["compact_sw"], sw[cy, cx])


def _p2p_full_worker(rank, world, port, r, steps, q):
    """C5 at full size: ranks share one B200; the compact state is generated on the device
    (seeded), non-owned cells poisoned; returns this rank's tiles' result digest parts."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2004_13475_b200 import nbb
    from paper_2004_13475_b200.shard import P2PCompactCA, ShardPlan
    plan = ShardPlan(r=r, rho=32, world=world, rank=rank, state="compact")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1700 + r)
    init = torch.randint(0, 2, (3 ** r,), dtype=torch.int64, device="cuda", generator=gen)
    own = torch.zeros(3 ** r, dtype=torch.bool, device="cuda")
    for o, c in plan.compact_segments():
        own[o:o + c] = True
    init[~own] = 7
    ca = P2PCompactCA(plan, dist, device=0, timeout_ms=120000)
    ca.load(init)
    ca.run(nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2), nbb.CaRule(), steps,
           torch.cuda.current_stream().cuda_stream)
    ca.check(torch.cuda.current_stream().cuda_stream)
    out = torch.where(own, ca.state(), torch.zeros_like(ca.state())).cpu()
    ca.close()
    dist.all_reduce(out)
    if rank == 0:
        q.put(out.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("r,world", [(17, 2), (18, 2)])
def test_p2p_compact_ca_full_size_r17(r, world):
    """C5 (n = 2^17, and 2^18) through the multi-rank P2P step loop (2 ranks time-sharing one B200,
    their non-owned cells poisoned) equals the single-GPU compact step loop bit for bit."""
    from paper_2004_13475_b200 import device as dev
    from paper_2004_13475_b200 import nbb
    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_full_worker, args=(i, world, port, r, steps, q)) for i in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=900)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1700 + r)
    a = torch.randint(0, 2, (3 ** r,), dtype=torch.int64, device="cuda", generator=gen)
    b = torch.empty_like(a)
    dev.ca_compact_run_dev(nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2), a.data_ptr(),
                           b.data_ptr(), steps, nbb.CaRule(), torch.cuda.current_stream().cuda_stream)
    want = (b if steps % 2 else a).cpu().numpy()
    assert np.array_equal(got, want)
