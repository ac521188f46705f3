"""Multi-GPU partition of the λ(ω) launch (one process per GPU).

The tile ordinal range o = ωy*W + ωx of the λ orthotope is split into contiguous
chunks, chunk = ceil(total / world) — the same split the reference applies to its
worker threads (dispatch.cpp:419-427); for the compact state rounded up to whole cluster
columns (compact_shard_chunk), the unit of the library's cluster pass. SW and RD need no exchange (RD ends in one
all-reduce of an int64). A CA step reads, besides its own tile, at most 8 cells of
neighbouring tiles (the tile's "halo"):

    (-1,-1) (0,-1) (1,-1) (-1,ρ-1) (ρ,ρ-2) (ρ,ρ-1) (ρ,ρ) (0,ρ)   (tile-local x, y)

Those owned by another rank are exchanged before every step: the static send/recv
lists are computed once here (host logic, numpy), packed/unpacked by the library's
gather/scatter kernels and moved by one NCCL all_to_all_single. Every rank keeps a
full replica of the embedded grid (identical addresses on every rank), of which it
only reads its own tiles plus the received halo cells.

state="compact" partitions the λ-ordered compact CA state (ρ = 32 tiles) instead: the
tiles are taken in the compact kernel's order u = ωx_b·H_b + ωy_b (a contiguous u range
is a contiguous slab of compact rows), and the exchanged indices are compact offsets
ωy·W + ωx of the halo cells (λ⁻¹ at full level). Same chunk rule, same ≤ 8 cells per tile.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

HALO = np.array([(-1, -1), (0, -1), (1, -1), (-1, -2), (-2, -3), (-2, -2), (-2, -1), (0, -1)],
                dtype=np.int64)


def compact_shard_chunk(r_b: int, tiles: int, Hb: int, world: int) -> int:
    """Tiles per rank of the compact-state CA (nbbhost::compact_shard_chunk): ceil(tiles / world)
    — the reference's contiguous worker chunks (dispatch.cpp:419-427) — rounded up to whole
    cluster columns of 9·Hb tiles when r_b >= 3, so every rank owns whole level-3 clusters (the
    batches of the library's cluster pass). Results are identical for any split."""
    world = max(1, world)
    if r_b >= 3 and Hb % 3 == 0 and tiles % (9 * Hb) == 0:
        col = 9 * Hb
        return -(-(tiles // col) // world) * col
    return -(-tiles // world)


def _halo_offsets(rho: int) -> np.ndarray:
    """The 8 candidate halo cells of a member tile, tile-local (x, y)."""
    return np.array([(-1, -1), (0, -1), (1, -1), (-1, rho - 1), (rho, rho - 2), (rho, rho - 1),
                     (rho, rho), (0, rho)], dtype=np.int64)


def _xy_digits(v: np.ndarray):
    """X(v), Y(v) of SURVEY App. A.1: bit 2j set iff base-3 digit j is 2 (X) / >= 1 (Y)."""
    v = v.astype(np.int64).copy()
    X = np.zeros_like(v)
    Y = np.zeros_like(v)
    j = 0
    while np.any(v):
        d = v % 3
        X |= (d == 2).astype(np.int64) << (2 * j)
        Y |= (d >= 1).astype(np.int64) << (2 * j)
        v //= 3
        j += 1
    return X, Y


def lambda_blocks(ordinals: np.ndarray, W: int):
    """λ(ω) of block ordinals (block_map.cpp:77-111 in closed form)."""
    ox, oy = ordinals % W, ordinals // W
    Xx, Yx = _xy_digits(ox)
    Xy, Yy = _xy_digits(oy)
    return Xx | (Xy << 1), Yx | (Yy << 1)


def lambda_inverse_blocks(bx: np.ndarray, by: np.ndarray, r_b: int, W: int) -> np.ndarray:
    """Ordinal of member blocks (λ⁻¹, block_map.cpp:113-148, gasket H table)."""
    ox = np.zeros_like(bx)
    oy = np.zeros_like(by)
    for mu in range(r_b, 0, -1):
        cx = (bx >> (mu - 1)) & 1
        cy = (by >> (mu - 1)) & 1
        beta = cx + cy  # (0,0)->0, (0,1)->1, (1,1)->2; (1,0) is not a member
        d = 3 ** ((mu + 1) // 2 - 1)
        if mu % 2 == 1:
            ox += beta * d
        else:
            oy += beta * d
    return oy * W + ox


@dataclass
class ShardPlan:
    r: int
    rho: int
    world: int
    rank: int
    total: int = 0
    chunk: int = 0
    begin: int = 0
    count: int = 0
    send_idx: np.ndarray = field(default=None, repr=False)   # flat cell indices, grouped by dest
    send_counts: list = field(default=None)
    recv_idx: np.ndarray = field(default=None, repr=False)   # grouped by source
    recv_counts: list = field(default=None)
    state: str = "embedded"   # or "compact" (λ-ordered CompactGrid CA state, ρ = 32)
    _dev: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        if self.state not in ("embedded", "compact"):
            raise ValueError(f"unknown state '{self.state}'")
        if self.state == "compact" and self.rho != 32:
            raise ValueError("the compact CA state uses rho = 32 tiles")
        rt = self.rho.bit_length() - 1
        self.r_b = self.r - rt
        self.W = 3 ** ((self.r_b + 1) // 2)
        self.Hb = 3 ** (self.r_b // 2)
        self.total = 3 ** self.r_b
        self.chunk = (compact_shard_chunk(self.r_b, self.total, self.Hb, self.world)
                      if self.state == "compact" else -(-self.total // self.world))
        self.begin = min(self.rank * self.chunk, self.total)
        self.count = max(0, min(self.chunk, self.total - self.begin))
        if self.world > 1:
            self._build_halo_lists()
        else:
            self.send_idx = self.recv_idx = np.zeros(0, dtype=np.int64)
            self.send_counts = self.recv_counts = [0]

    def owner(self, ordinals: np.ndarray) -> np.ndarray:
        return ordinals // self.chunk

    def ordinal_of_tile(self, t: np.ndarray) -> np.ndarray:
        """Block ordinal ωy_b·W + ωx_b of tile ids in this plan's order."""
        if self.state == "compact":
            return (t % self.Hb) * self.W + t // self.Hb
        return t

    def tile_of_ordinal(self, o: np.ndarray) -> np.ndarray:
        if self.state == "compact":
            return (o % self.W) * self.Hb + o // self.W
        return o

    def owned_blocks(self):
        """(bx, by) block coordinates of this rank's tiles."""
        t = np.arange(self.begin, self.begin + self.count, dtype=np.int64)
        return lambda_blocks(self.ordinal_of_tile(t), self.W)

    def halo_owner_table(self) -> np.ndarray:
        """uint8 [tiles * 8]: the rank owning each tile's k-th halo cell (0 where the cell is
        not a member) — the table the P2P compact CA kernel selects peer buffers with."""
        n, rho = 1 << self.r, self.rho
        t = np.arange(self.total, dtype=np.int64)
        bx, by = lambda_blocks(self.ordinal_of_tile(t), self.W)
        off = _halo_offsets(rho)
        cx = (bx * rho)[:, None] + off[None, :, 0]
        cy = (by * rho)[:, None] + off[None, :, 1]
        ok = (cx >= 0) & (cy >= 0) & (cx < n) & (cy < n)
        ok &= (np.where(ok, cx, 0) & (n - 1 - np.where(ok, cy, 0))) == 0
        own = np.zeros(cx.shape, dtype=np.int64)
        own[ok] = self.owner(self.tile_of_ordinal(
            lambda_inverse_blocks(cx[ok] // rho, cy[ok] // rho, self.r_b, self.W)))
        return own.astype(np.uint8).ravel()

    def _build_halo_lists(self):
        n, rho = 1 << self.r, self.rho
        t = np.arange(self.total, dtype=np.int64)
        bx, by = lambda_blocks(self.ordinal_of_tile(t), self.W)
        off = _halo_offsets(rho)
        cx = (bx * rho)[:, None] + off[None, :, 0]
        cy = (by * rho)[:, None] + off[None, :, 1]
        needer = np.broadcast_to(self.owner(t)[:, None], cx.shape)
        ok = (cx >= 0) & (cy >= 0) & (cx < n) & (cy < n)
        cx, cy, needer = cx[ok], cy[ok], needer[ok]
        memb = (cx & (n - 1 - cy)) == 0
        cx, cy, needer = cx[memb], cy[memb], needer[memb]
        own_t = self.tile_of_ordinal(lambda_inverse_blocks(cx // rho, cy // rho, self.r_b, self.W))
        src = self.owner(own_t)
        remote = src != needer
        if self.state == "compact":  # compact offset ωy·W + ωx of the cell
            flat = lambda_inverse_blocks(cx[remote], cy[remote], self.r, 3 ** ((self.r + 1) // 2))
        else:
            flat = (cy * n + cx)[remote]
        src, needer = src[remote], needer[remote]
        # unique (needer, src, cell) triples in a canonical order both sides agree on
        key = np.unique(np.stack([needer, src, flat], axis=1), axis=0)
        self.all_pairs = key
        mine_recv = key[key[:, 0] == self.rank]
        mine_send = key[key[:, 1] == self.rank]
        self.recv_counts = [int(np.sum(mine_recv[:, 1] == p)) for p in range(self.world)]
        self.send_counts = [int(np.sum(mine_send[:, 0] == p)) for p in range(self.world)]
        # recv grouped by source rank (key sorted by needer, src, flat)
        self.recv_idx = mine_recv[:, 2].copy()
        # send grouped by destination: order by (needer, src=me, flat)
        self.send_idx = mine_send[np.lexsort((mine_send[:, 2], mine_send[:, 0]))][:, 2].copy()

    def halo_cells_received(self) -> int:
        return int(sum(self.recv_counts))

    def compact_segments(self):
        """(offset, count) runs of the compact state holding this rank's tiles (state="compact"):
        the same decomposition the library's compact RD / SW use (nbb_capi.cu compact_segments):
        a tile u = ωx_b·H_b + ωy_b is 9 compact rows x 27 columns, a tile row 9 full rows."""
        W = 27 * self.Hb
        segs, u, e = [], self.begin, self.begin + self.count
        while u < e:
            wxb, c0 = divmod(u, self.Hb)
            if c0 == 0 and e - u >= self.Hb:
                k = (e - u) // self.Hb
                segs.append((9 * wxb * W, 9 * W * k))
                u += k * self.Hb
            else:
                c1 = min(self.Hb, c0 + (e - u))
                segs += [((9 * wxb + row) * W + 27 * c0, 27 * (c1 - c0)) for row in range(9)]
                u += c1 - c0
        return segs

    def local_config(self, config):
        """The launch config restricted to this rank's chunk of block ordinals."""
        import copy
        c = copy.copy(config)
        c.shard_begin = self.begin
        c.shard_count = max(self.count, 0)
        if self.count == 0:
            c.shard_begin, c.shard_count = self.total, 1  # empty launch
        return c

    # ---- exchange -----------------------------------------------------------------
    def exchange_halo(self, grid, dist, gather: Optional[Callable] = None,
                      scatter: Optional[Callable] = None, group=None):
        """Bring this rank's remote halo cells up to date in `grid` (a torch tensor)."""
        if self.world == 1:
            return
        import torch
        key = (grid.device, grid.dtype)
        if key not in self._dev:
            self._dev[key] = (torch.from_numpy(self.send_idx).to(grid.device),
                              torch.from_numpy(self.recv_idx).to(grid.device))
        sidx, ridx = self._dev[key]
        flat = grid.view(-1)
        if gather is None:
            gather = _kernel_gather
        if scatter is None:
            scatter = _kernel_scatter
        send = gather(flat, sidx)
        recv = torch.empty(int(sum(self.recv_counts)), dtype=grid.dtype, device=grid.device)
        if grid.is_cuda and dist.get_backend(group) == "gloo":
            # ranks sharing one GPU (test setups): stage the tiny halo through host memory
            send_h, recv_h = send.cpu(), recv.cpu()
            dist.all_to_all_single(recv_h, send_h, output_split_sizes=self.recv_counts,
                                   input_split_sizes=self.send_counts, group=group)
            recv.copy_(recv_h)
        else:
            dist.all_to_all_single(recv, send, output_split_sizes=self.recv_counts,
                                   input_split_sizes=self.send_counts, group=group)
        scatter(flat, ridx, recv)


def sharded_reduction(plan: ShardPlan, config, d_state: int, dist, stream: int = 0,
                      device: int = 0) -> int:
    """run_reduction over the shards (dispatch.cpp:490-515): each rank sums its own tiles on its
    GPU (embedded grid: the tile kernels on cfg.shard_*; compact state: the segments of its
    tiles), then ONE int64 all-reduce (NCCL; gloo when ranks share a GPU) — the final reduction.
    int64 addition wraps like the reference's, so the partial sums add up exactly."""
    import torch
    from . import device as dev
    c = plan.local_config(config)
    part, host = _scalar_buffers(device)  # the kernels overwrite the device scalar (no zero-fill)
    if plan.state == "compact":
        dev.reduction_compact_dev(c, d_state, part.data_ptr(), stream)
    else:
        dev.reduction_dev(c, d_state, part.data_ptr(), stream)
    ts = (torch.cuda.ExternalStream(stream, device=part.device) if stream
          else torch.cuda.default_stream(part.device))
    with torch.cuda.stream(ts):
        if plan.world > 1:
            if dist.get_backend() == "nccl":
                dist.all_reduce(part)
            else:
                h = part.cpu()
                dist.all_reduce(h)
                return int(h.item())
        host.copy_(part, non_blocking=True)
        ts.synchronize()
    return int(host[0])


_SCALARS: dict = {}


def _scalar_buffers(device: int):
    """One int64 device scalar and one pinned host scalar per device, reused across calls."""
    import torch
    b = _SCALARS.get(device)
    if b is None:
        b = (torch.empty(1, dtype=torch.int64, device=torch.device("cuda", device)),
             torch.empty(1, dtype=torch.int64, pin_memory=True))
        _SCALARS[device] = b
    return b


def sharded_single_write(plan: ShardPlan, config, d_state: int, stream: int = 0) -> None:
    """run_single_write over the shards: each rank writes its own tiles; no exchange."""
    from . import device as dev
    c = plan.local_config(config)
    if plan.state == "compact":
        dev.single_write_compact_dev(c, d_state, stream)
    else:
        dev.single_write_dev(c, d_state, stream)


def _cfg_for(t):
    from .nbb import DispatchConfig
    return DispatchConfig(cell_width=t.element_size(), device=t.device.index or 0)


def _kernel_gather(flat, idx):
    import torch
    from . import device as dev
    out = torch.empty(idx.numel(), dtype=flat.dtype, device=flat.device)
    if idx.numel():
        from .nbb import _check, _lib
        import ctypes
        c = _cfg_for(flat).to_c()
        _check(_lib().nbb_gpu_gather_cells_dev(ctypes.byref(c), ctypes.c_void_p(flat.data_ptr()),
                                               ctypes.c_void_p(idx.data_ptr()), idx.numel(),
                                               ctypes.c_void_p(out.data_ptr()),
                                               ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out


def _kernel_scatter(flat, idx, vals):
    if idx.numel() == 0:
        return
    import ctypes
    import torch
    from .nbb import _check, _lib
    c = _cfg_for(flat).to_c()
    _check(_lib().nbb_gpu_scatter_cells_dev(ctypes.byref(c), ctypes.c_void_p(flat.data_ptr()),
                                            ctypes.c_void_p(idx.data_ptr()), idx.numel(),
                                            ctypes.c_void_p(vals.data_ptr()),
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))


# ---- the compact CA over peer memory (one kernel per step, no separate exchange) ----------
class _DevArray:
    """A raw device allocation seen by torch (zero-copy, __cuda_array_interface__)."""

    def __init__(self, ptr: int, count: int, typestr: str = "<i8"):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


class P2PUnavailable(RuntimeError):
    """CUDA IPC peer mappings could not be opened on every rank (raised on all ranks alike)."""


class P2PCompactCA:
    """Multi-GPU compact CA where the exchange lives inside the step kernel.

    Every rank allocates its two compact buffers and a 16-byte sync word with cudaMalloc
    (nbb_gpu_malloc), exports them as CUDA IPC handles, opens every peer's (one
    all_gather_object at setup), and then runs each step as ONE launch of
    nbb_gpu_ca_compact_p2p_dev (the step loop in C++): each kernel waits until all ranks
    finished the previous step, reads the ≤ 8 halo cells per tile that other ranks own
    straight from their buffers (NVLink loads through the IPC mappings), writes its own tiles,
    and its last CTA adds one arrival to every rank's counter. No host synchronisation and
    no collective inside the step loop; the NCCL `exchange_halo` path is the baseline.
    """

    def __init__(self, plan: ShardPlan, dist, device: int = 0, timeout_ms: int = 20000,
                 two_step: bool = True):
        import ctypes
        import torch
        from . import _abi
        if plan.state != "compact":
            raise ValueError("P2PCompactCA needs ShardPlan(state='compact')")
        if plan.world > 8:
            raise ValueError("P2PCompactCA supports up to 8 ranks")
        self.plan, self.device, self.timeout_ms, self.dist = plan, device, timeout_ms, dist
        self.two_step = two_step  # passes of two steps (ca_compact2_kernel) vs one launch per step
        self.lib = lib = _abi.load()
        self.count = 3 ** plan.r
        nbytes = self.count * 8

        def alloc(b):
            p = ctypes.c_void_p()
            _check(lib.nbb_gpu_malloc(device, b, ctypes.byref(p)))
            return p.value

        self._own = [alloc(nbytes), alloc(nbytes), alloc(16)]   # buffer 0, buffer 1, sync
        handles = []
        for ptr in self._own:
            h = (ctypes.c_uint8 * 64)()
            _check(lib.nbb_gpu_ipc_handle(device, ctypes.c_void_p(ptr), h))
            handles.append(bytes(h))
        gathered = [None] * plan.world
        dist.all_gather_object(gathered, handles)
        self._opened = []
        peers = []
        err = None
        try:
            for r, hs in enumerate(gathered):
                if r == plan.rank:
                    peers.append(self._own)
                    continue
                ptrs = []
                for h in hs:
                    p = ctypes.c_void_p()
                    _check(lib.nbb_gpu_ipc_open(device, (ctypes.c_uint8 * 64).from_buffer_copy(h),
                                                ctypes.byref(p)))
                    ptrs.append(p.value)
                    self._opened.append(p.value)
                peers.append(ptrs)
        except Exception as e:  # noqa: BLE001 - agreed on below, raised on every rank
            err = e
        # every rank must agree, or one rank would wait in a step kernel for a peer that gave up
        ok = torch.tensor([0 if err else 1], dtype=torch.int32,
                          device=torch.device("cuda", device) if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            for ptr in self._opened:
                lib.nbb_gpu_ipc_close(device, ctypes.c_void_p(ptr))
            for ptr in self._own:
                lib.nbb_gpu_free(device, ctypes.c_void_p(ptr))
            self._opened, self._own = [], []
            raise P2PUnavailable(f"peer mappings unavailable on some rank ({err or 'another rank'})")
        dev = torch.device("cuda", device)
        self._peer_buf = [torch.tensor([peers[r][b] for r in range(plan.world)], dtype=torch.int64,
                                       device=dev) for b in (0, 1)]
        self._peer_flag = torch.tensor([peers[r][2] for r in range(plan.world)], dtype=torch.int64,
                                       device=dev)
        self.buffers = [torch.as_tensor(_DevArray(p, self.count), device=dev) for p in self._own[:2]]
        self._args = _abi.NbbP2P(plan.world, plan.rank, (ctypes.c_void_p * 2)(*self._own[:2]),
                                 (ctypes.c_void_p * 2)(*(t.data_ptr() for t in self._peer_buf)),
                                 None, self._own[2], self._peer_flag.data_ptr(),
                                 timeout_ms)
        self.step_index = 0
        self.pass_index = 0  # passes (launches) run so far: the state lives in buffer pass_index & 1

    def load(self, compact_state) -> None:
        """Set the state (a (3^r,) int64 tensor; this rank's tiles must be current). Collective:
        every rank loads before any rank's first step reads a peer. Call once, before the
        first step (the device step counter starts at 0)."""
        import torch
        if self.step_index:
            raise RuntimeError("P2PCompactCA.load: the step sequence has already started")
        self.buffers[0].copy_(compact_state.to(self.buffers[0].device).view(-1))
        torch.cuda.synchronize(self.device)
        self.dist.barrier()

    def state(self):
        """The current state buffer (this rank's tiles are current)."""
        return self.buffers[self.pass_index & 1]

    def run(self, config, rule, steps: int, stream) -> None:
        """`steps` steps issued back to back by the library: passes of up to config.pass_steps
        steps (default 4; nbb_gpu_pass_plan names them), or one kernel per step with
        two_step=False."""
        import ctypes
        local = self.plan.local_config(config)
        c = local.to_c()
        fn = (self.lib.nbb_gpu_ca_compact_p2p_passes_dev if self.two_step
              else self.lib.nbb_gpu_ca_compact_p2p_dev)
        _check(fn(ctypes.byref(c), self.pass_index, steps, rule.birth, rule.survive,
                  ctypes.byref(self._args), ctypes.c_void_p(stream)))
        self.step_index += steps
        if self.two_step:
            from . import _abi
            st = _abi.NbbPassStats()
            _check(self.lib.nbb_gpu_pass_plan(ctypes.byref(c), steps, 0, ctypes.byref(st)))
            self.pass_index += st.passes
        else:
            self.pass_index += steps

    def step(self, config, rule, stream) -> None:
        self.run(config, rule, 1, stream)

    def check(self, stream) -> None:
        """Raise if any step timed out waiting for the other ranks (synchronises)."""
        import ctypes
        _check(self.lib.nbb_gpu_p2p_check(ctypes.byref(self._args), ctypes.c_void_p(stream)))

    def close(self) -> None:
        """Collective: no rank unmaps or frees while a peer's step may still read it."""
        import ctypes
        import torch
        torch.cuda.synchronize(self.device)
        self.dist.barrier()
        for p in self._opened:
            self.lib.nbb_gpu_ipc_close(self.device, ctypes.c_void_p(p))
        self._opened = []
        self.buffers = []
        self.dist.barrier()
        for p in self._own:
            self.lib.nbb_gpu_free(self.device, ctypes.c_void_p(p))
        self._own = []


def _check(rc: int) -> None:
    from .nbb import _check as check
    check(rc)


class NcclCompactCA:
    """The multi-process compact CA over the library's own NCCL communicator (nbb_gpu_comm_*,
    include/nbb_gpu.h): one process per GPU, rank i owning the contiguous tile chunk i of
    compact_shard_chunk (dispatch.cpp:419-427); before every pass of up to 8 steps the halo cells
    its tiles read from other ranks within 8 steps are exchanged by ncclSend / ncclRecv inside the
    library, then the pass kernel advances the rank's tiles. The communicator's id travels over
    the caller's process group (`dist`, any backend); dist=None is a single rank."""

    def __init__(self, r: int, dist=None, device: int = 0):
        import ctypes
        import torch
        from . import _abi
        self.lib = lib = _abi.load()
        self.r, self.device = r, device
        self.world = dist.get_world_size() if dist is not None else 1
        self.rank = dist.get_rank() if dist is not None else 0
        uid = (ctypes.c_uint8 * 128)()
        if self.rank == 0:
            _check(lib.nbb_gpu_comm_unique_id(uid))
        if dist is not None:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0)
            uid = (ctypes.c_uint8 * 128).from_buffer_copy(box[0])
        self._comm = ctypes.c_void_p()
        _check(lib.nbb_gpu_comm_init(uid, self.world, self.rank, device, ctypes.byref(self._comm)))
        dev = torch.device("cuda", device)
        self.buffers = [torch.zeros(3 ** r, dtype=torch.int64, device=dev) for _ in range(2)]
        self.cur = 0
        self.passes = 0

    def load(self, compact_state) -> None:
        """Set the state (a (3^r,) int64 tensor; this rank's tiles must be current)."""
        self.buffers[0].copy_(compact_state.to(self.buffers[0].device).view(-1))
        self.cur = 0

    def state(self):
        return self.buffers[self.cur]

    def run(self, config, rule, steps: int, stream) -> None:
        import ctypes
        from . import _abi
        st = _abi.NbbPassStats()
        a, b = self.buffers[self.cur], self.buffers[self.cur ^ 1]
        _check(self.lib.nbb_gpu_ca_compact_comm_dev(ctypes.byref(config.to_c()), self._comm,
                                                    ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                                                    steps, rule.birth, rule.survive, ctypes.c_void_p(stream),
                                                    ctypes.byref(st)))
        self.cur ^= st.result_in_b
        self.passes += st.passes

    def reduction(self, config, stream) -> int:
        """run_reduction of the current state: the rank's partial sum + one ncclAllReduce."""
        import ctypes
        import torch
        out = torch.empty(1, dtype=torch.int64, device=self.buffers[0].device)
        _check(self.lib.nbb_gpu_reduction_compact_comm_dev(ctypes.byref(config.to_c()), self._comm,
                                                           ctypes.c_void_p(self.state().data_ptr()),
                                                           ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream)))
        torch.cuda.synchronize(self.device)
        return int(out.item())

    def close(self) -> None:
        if self._comm:
            _check(self.lib.nbb_gpu_comm_destroy(self._comm))
            self._comm = None
