"""Multi-GPU partition of the λ(ω) launch (one process per GPU).

The tile ordinal range o = ωy*W + ωx of the λ orthotope is split into contiguous
chunks, chunk = ceil(total / world) — the same split the reference applies to its
worker threads (dispatch.cpp:419-427). SW and RD need no exchange (RD ends in one
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
        self.chunk = -(-self.total // self.world)
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
