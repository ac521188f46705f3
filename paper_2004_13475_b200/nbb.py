"""Host-side mirror of the reference's public API (namespace nbb), backed by the
sm_100a library through the C ABI (include/nbb_gpu.h).

Same names, argument meaning and error behaviour as
/root/reference/proj/include/nbb/{fractal,dispatch}.hpp, so code written
against the reference reads the same:

    cfg = DispatchConfig(r=10, rho=32, mode=MapMode.Lambda)
    sw = run_single_write(cfg)              # dispatch.cpp:481-488
    rd = run_reduction(cfg, grid)           # dispatch.cpp:490-515
    ca = run_ca(cfg, grid, steps, CaRule()) # dispatch.cpp:517-557

Exceptions mirror the reference's std:: types: InvalidArgument (ValueError) for
std::invalid_argument, OutOfRange (IndexError), ResourceError, DomainError,
OverflowError_ and CudaError (no device / CUDA failure: there is no CPU fallback).
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi


# ---- exceptions ----------------------------------------------------------------
class NbbError(Exception):
    pass


class InvalidArgument(NbbError, ValueError):
    pass


class OutOfRange(NbbError, IndexError):
    pass


class ResourceError(NbbError, RuntimeError):
    pass


class CudaError(NbbError, RuntimeError):
    pass


class DomainError(NbbError, ValueError):
    pass


class OverflowError_(NbbError, OverflowError):
    pass


class KernelError(NbbError, RuntimeError):
    pass


_EXC = {
    _abi.ERR_INVALID_ARGUMENT: InvalidArgument,
    _abi.ERR_OUT_OF_RANGE: OutOfRange,
    _abi.ERR_RESOURCE: ResourceError,
    _abi.ERR_CUDA: CudaError,
    _abi.ERR_NCCL: CudaError,
    _abi.ERR_DOMAIN: DomainError,
    _abi.ERR_OVERFLOW: OverflowError_,
    _abi.ERR_RUNTIME: KernelError,
}


def _lib():
    return _abi.load()


def _check(rc: int) -> None:
    if rc != _abi.OK:
        msg = _lib().nbb_gpu_last_error().decode(errors="replace")
        raise _EXC.get(rc, NbbError)(msg)


# ---- enums (dispatch.hpp:16-17, block_map.hpp:46-50) -----------------------------
class MapMode(enum.IntEnum):
    BoundingBox = _abi.MODE_BB
    Lambda = _abi.MODE_LAMBDA


class IntraBlockStrategy(enum.IntEnum):
    FurtherUnrolling = _abi.STRATEGY_UNROLL
    SharedLookupTable = _abi.STRATEGY_LUT
    BoundingSubBoxes = _abi.STRATEGY_SUBBOX


class LambdaBackend(enum.IntEnum):
    Direct = _abi.BACKEND_DIRECT
    MmaV1 = _abi.BACKEND_MMA1
    MmaV2 = _abi.BACKEND_MMA2
    MmaV3 = _abi.BACKEND_MMA3


class KernelFamily(enum.IntEnum):
    """Device implementation choice (not in the reference)."""
    Auto = _abi.KERNEL_AUTO
    PerCell = _abi.KERNEL_PERCELL
    Tile = _abi.KERNEL_TILE


_MODE_NAMES = {"bb": MapMode.BoundingBox, "lambda": MapMode.Lambda}
_STRATEGY_NAMES = {"unroll": IntraBlockStrategy.FurtherUnrolling,
                   "lut": IntraBlockStrategy.SharedLookupTable,
                   "subbox": IntraBlockStrategy.BoundingSubBoxes}
_BACKEND_NAMES = {"direct": LambdaBackend.Direct, "mma1": LambdaBackend.MmaV1,
                  "mma2": LambdaBackend.MmaV2, "mma3": LambdaBackend.MmaV3}


def mode_from_string(name: str) -> MapMode:            # dispatch.cpp:25-29
    if name not in _MODE_NAMES:
        raise InvalidArgument(f"unknown mode '{name}' (expected bb or lambda)")
    return _MODE_NAMES[name]


def strategy_from_string(name: str) -> IntraBlockStrategy:  # block_map.cpp:166-172
    if name not in _STRATEGY_NAMES:
        raise InvalidArgument(f"unknown strategy '{name}' (expected unroll, lut or subbox)")
    return _STRATEGY_NAMES[name]


def backend_from_string(name: str) -> LambdaBackend:   # dispatch.cpp:41-48
    if name not in _BACKEND_NAMES:
        raise InvalidArgument(f"unknown backend '{name}' (expected direct, mma1, mma2 or mma3)")
    return _BACKEND_NAMES[name]


def to_string(v) -> str:
    for table in (_MODE_NAMES, _STRATEGY_NAMES, _BACKEND_NAMES):
        for k, e in table.items():
            if e is v:
                return k
    raise InvalidArgument(f"unknown enumerator {v!r}")


# ---- FractalSpec (fractal.hpp:53-102) --------------------------------------------
@dataclass(frozen=True)
class FractalSpec:
    name: str
    k: int
    s: int
    offsets: tuple

    @staticmethod
    def sierpinski() -> "FractalSpec":
        return FractalSpec("sierpinski", 3, 2, ((0, 0), (0, 1), (1, 1)))

    @staticmethod
    def vicsek() -> "FractalSpec":
        return FractalSpec("vicsek", 5, 3, ((1, 1), (1, 0), (1, 2), (0, 1), (2, 1)))

    @staticmethod
    def carpet() -> "FractalSpec":
        return FractalSpec("carpet", 8, 3, ((0, 0), (1, 0), (2, 0), (0, 1), (2, 1), (0, 2),
                                            (1, 2), (2, 2)))

    @staticmethod
    def builtin(name: str) -> "FractalSpec":
        table = {"sierpinski": FractalSpec.sierpinski, "vicsek": FractalSpec.vicsek,
                 "carpet": FractalSpec.carpet}
        if name not in table:
            raise InvalidArgument(f"unknown builtin fractal '{name}'")
        return table[name]()

    def replica_count(self) -> int:
        return self.k

    def scale_factor(self) -> int:
        return self.s

    def side_length(self, level: int) -> int:
        if level < 0:
            raise InvalidArgument("checked_pow: negative exponent")
        return self.s ** level

    def volume(self, level: int) -> int:
        return self.k ** level

    def orthotope_dims(self, level: int):
        if level < 0:
            raise InvalidArgument("orthotope_dims: negative level")
        return self.k ** ((level + 1) // 2), self.k ** (level // 2)

    def to_c(self) -> _abi.NbbSpec:
        c = _abi.NbbSpec()
        c.name = self.name.encode()[:31]
        c.k = self.k
        c.s = self.s
        for i, (x, y) in enumerate(self.offsets[:_abi.MAX_REPLICAS]):  # k > 9 fails validation
            c.offset_x[i] = x
            c.offset_y[i] = y
        return c


# ---- DispatchConfig (dispatch.hpp:25-38) -----------------------------------------
@dataclass
class DispatchConfig:
    spec: FractalSpec = field(default_factory=FractalSpec.sierpinski)
    r: int = 0
    rho: int = 1
    mode: MapMode = MapMode.Lambda
    strategy: IntraBlockStrategy = IntraBlockStrategy.BoundingSubBoxes
    backend: LambdaBackend = LambdaBackend.Direct
    workers: int = 1
    timing: bool = False
    max_cells: int = 1 << 24
    # device-side extensions
    cell_width: int = 8
    kernel: KernelFamily = KernelFamily.Auto
    device: int = 0
    shard_begin: int = 0
    shard_count: int = 0  # 0 = every block ordinal of the plan
    flags: int = 0        # _abi.FLAG_* (e.g. FLAG_OUT_ZEROED)
    pass_steps: int = 0   # compact CA: at most this many steps per pass (1..12; 0 = 8; above 8: r >= 8 only)

    def to_c(self) -> _abi.NbbConfig:
        c = _abi.NbbConfig()
        c.spec = self.spec.to_c()
        c.r = self.r
        c.rho = self.rho
        c.mode = int(self.mode)
        c.strategy = int(self.strategy)
        c.backend = int(self.backend)
        c.workers = self.workers
        c.timing = 1 if self.timing else 0
        c.cell_width = self.cell_width
        c.kernel = int(self.kernel)
        c.device = self.device
        c.max_cells = self.max_cells
        c.shard_begin = self.shard_begin
        c.shard_count = self.shard_count
        c.flags = self.flags
        c.pass_steps = self.pass_steps
        return c

    def validate(self) -> None:                         # dispatch.cpp:50-114
        _check(_lib().nbb_gpu_validate(ctypes.byref(self.to_c())))


# ---- WorkReport (dispatch.hpp:44-61) ---------------------------------------------
@dataclass
class WorkReport:
    spec_name: str = ""
    r: int = 0
    rho: int = 1
    mode: MapMode = MapMode.Lambda
    strategy: IntraBlockStrategy = IntraBlockStrategy.BoundingSubBoxes
    backend: LambdaBackend = LambdaBackend.Direct
    blocks_launched: int = 0
    threads_launched: int = 0
    threads_active: int = 0
    threads_wasted: int = 0
    map_ops: int = 0
    micros: int = 0
    map_levels: int = 0

    @staticmethod
    def from_c(c: _abi.NbbReport) -> "WorkReport":
        return WorkReport(c.spec_name.decode(), c.r, c.rho, MapMode(c.mode),
                          IntraBlockStrategy(c.strategy), LambdaBackend(c.backend),
                          c.blocks_launched, c.threads_launched, c.threads_active,
                          c.threads_wasted, c.map_ops, c.micros, c.map_levels)

    def to_c(self) -> _abi.NbbReport:
        c = _abi.NbbReport()
        c.spec_name = self.spec_name.encode()[:31]
        c.r, c.rho = self.r, self.rho
        c.mode, c.strategy, c.backend = int(self.mode), int(self.strategy), int(self.backend)
        c.map_levels = self.map_levels
        c.blocks_launched, c.threads_launched = self.blocks_launched, self.threads_launched
        c.threads_active, c.threads_wasted = self.threads_active, self.threads_wasted
        c.map_ops, c.micros = self.map_ops, self.micros
        return c

    @staticmethod
    def csv_header() -> str:
        return _lib().nbb_gpu_csv_header().decode()

    def csv_row(self) -> str:
        buf = ctypes.create_string_buffer(512)
        _check(_lib().nbb_gpu_report_csv_row(ctypes.byref(self.to_c()), buf, 512))
        return buf.value.decode()


# ---- Grid (dispatch.hpp:65-93) ---------------------------------------------------
class Grid:
    """Dense row-major embedded grid of int64 cells (index y*n + x)."""

    def __init__(self, spec: FractalSpec, r: int, values: Optional[np.ndarray] = None):
        n = spec.side_length(r)
        self.spec = spec
        self._r = r
        self._n = n
        self._generation = 0
        if values is None:
            values = np.zeros((n, n), dtype=np.int64)
        values = np.asarray(values)
        if values.dtype != np.int64 or values.shape != (n, n):
            raise InvalidArgument(f"grid values must be int64 of shape ({n}, {n})")
        self.values = np.ascontiguousarray(values)

    def level(self) -> int:
        return self._r

    def side(self) -> int:
        return self._n

    def generation(self) -> int:
        return self._generation

    def bump_generation(self) -> None:
        self._generation += 1

    def at(self, x: int, y: int) -> int:
        return int(self.values[y, x])

    def set(self, x: int, y: int, v: int) -> None:
        self.values[y, x] = v

    def copy(self) -> "Grid":
        g = Grid(self.spec, self._r, self.values.copy())
        g._generation = self._generation
        return g

    def __eq__(self, other) -> bool:
        return (isinstance(other, Grid) and self._r == other._r and self._n == other._n and
                np.array_equal(self.values, other.values))

    def _ptr(self):
        return self.values.ctypes.data_as(ctypes.c_void_p)


def random_member_grid(spec: FractalSpec, r: int, seed: int, modulus: int,
                       max_cells: int = 1 << 24) -> Grid:
    """dispatch.cpp:133-149, bit-identical (std::mt19937_64, row-major members)."""
    g = Grid(spec, r)
    _check(_lib().nbb_gpu_random_member_grid(ctypes.byref(spec.to_c()), r, seed, modulus,
                                             max_cells, g._ptr()))
    return g


def random_member_values(spec: FractalSpec, r: int, seed: int, modulus: int) -> np.ndarray:
    """The member values random_member_grid assigns, in row-major member order."""
    out = np.empty(spec.volume(r), dtype=np.int64)
    _check(_lib().nbb_gpu_random_member_values(ctypes.byref(spec.to_c()), r, seed, modulus,
                                                out.ctypes.data_as(ctypes.c_void_p)))
    return out


# ---- workloads ------------------------------------------------------------------
@dataclass
class SingleWriteResult:
    grid: Grid
    report: WorkReport


@dataclass
class ReductionResult:
    value: int
    report: WorkReport


@dataclass
class CaRule:                                             # dispatch.hpp:131-134
    birth: int = 1 << 3
    survive: int = (1 << 2) | (1 << 3)


@dataclass
class CaResult:
    grid: Grid
    reports: List[WorkReport]


def launch_block_count(config: DispatchConfig) -> int:   # dispatch.cpp:475-479
    out = ctypes.c_uint64()
    _check(_lib().nbb_gpu_launch_block_count(ctypes.byref(config.to_c()), ctypes.byref(out)))
    return out.value


def plan_report(config: DispatchConfig) -> WorkReport:
    rep = _abi.NbbReport()
    _check(_lib().nbb_gpu_plan_report(ctypes.byref(config.to_c()), ctypes.byref(rep)))
    return WorkReport.from_c(rep)


def run_single_write(config: DispatchConfig) -> SingleWriteResult:
    if config.r < 0:
        raise InvalidArgument("checked_pow: negative exponent")
    g = Grid(config.spec, config.r) if config.r <= 16 else None
    if g is None:
        raise ResourceError("host grid above r = 16 is not supported by the host-buffer API")
    rep = _abi.NbbReport()
    _check(_lib().nbb_gpu_single_write(ctypes.byref(config.to_c()), g._ptr(), ctypes.byref(rep)))
    return SingleWriteResult(g, WorkReport.from_c(rep))


def run_reduction(config: DispatchConfig, grid: Grid) -> ReductionResult:
    v = ctypes.c_int64()
    rep = _abi.NbbReport()
    _check(_lib().nbb_gpu_reduction(ctypes.byref(config.to_c()), grid._ptr(), grid.level(),
                                    ctypes.byref(v), ctypes.byref(rep)))
    return ReductionResult(v.value, WorkReport.from_c(rep))


def run_ca(config: DispatchConfig, initial: Grid, steps: int, rule: CaRule = CaRule()) -> CaResult:
    out = Grid(initial.spec, initial.level()) if initial.level() >= 0 else None
    reps = (_abi.NbbReport * max(steps, 1))()
    _check(_lib().nbb_gpu_ca(ctypes.byref(config.to_c()), initial._ptr(), initial.level(), steps,
                             rule.birth, rule.survive, out._ptr(), reps))
    out._generation = initial.generation() + steps
    return CaResult(out, [WorkReport.from_c(reps[i]) for i in range(steps)])


def _devices(devices) -> tuple:
    ds = [int(d) for d in devices]
    return (ctypes.c_int32 * len(ds))(*ds), len(ds)


def run_ca_multi(config: DispatchConfig, devices, initial: Grid, steps: int, rule: CaRule = CaRule()) -> CaResult:
    """run_ca with the reference's workers mapped to `devices` of this process (nbb_gpu_ca_multi):
    contiguous chunks of the compact tile range, halos over peer memory; byte-identical for any
    device list (devices may repeat)."""
    arr, nd = _devices(devices)
    out = Grid(initial.spec, initial.level())
    reps = (_abi.NbbReport * max(steps, 1))()
    _check(_lib().nbb_gpu_ca_multi(ctypes.byref(config.to_c()), arr, nd, initial._ptr(), initial.level(), steps,
                                   rule.birth, rule.survive, out._ptr(), reps))
    out._generation = initial.generation() + steps
    return CaResult(out, [WorkReport.from_c(reps[i]) for i in range(steps)])


def run_reduction_multi(config: DispatchConfig, devices, grid: Grid) -> ReductionResult:
    """run_reduction with one worker (contiguous tile chunk) per entry of `devices`."""
    arr, nd = _devices(devices)
    v = ctypes.c_int64()
    rep = _abi.NbbReport()
    _check(_lib().nbb_gpu_reduction_multi(ctypes.byref(config.to_c()), arr, nd, grid._ptr(), grid.level(),
                                          ctypes.byref(v), ctypes.byref(rep)))
    return ReductionResult(v.value, WorkReport.from_c(rep))


def work_quotient(bounding_box: WorkReport, lam: WorkReport, weighted: bool = False) -> float:
    q = ctypes.c_double()
    _check(_lib().nbb_gpu_work_quotient(ctypes.byref(bounding_box.to_c()), ctypes.byref(lam.to_c()),
                                        1 if weighted else 0, ctypes.byref(q)))
    return q.value


def lambda_coords(config: DispatchConfig, level: int) -> np.ndarray:
    """λ(ω) of every ω of the level orthotope, shape (W*H, 2), ordinal-major."""
    w, h = config.spec.orthotope_dims(level)
    out = np.empty((w * h, 2), dtype=np.int64)
    _check(_lib().nbb_gpu_lambda_coords(ctypes.byref(config.to_c()), level,
                                        out.ctypes.data_as(ctypes.c_void_p)))
    return out


# ---- compact codec (block_map.hpp:82-132) ------------------------------------------
class CompactGrid:
    """k^level values row-major over the packing orthotope (x fastest): value(ω) =
    embedded(λ(ω)). `values` is a (height, width) int64 array."""

    def __init__(self, spec: FractalSpec, level: int, values: Optional[np.ndarray] = None):
        w, h = spec.orthotope_dims(level)
        self.spec, self._level, self._w, self._h = spec, level, w, h
        if values is None:
            values = np.zeros((h, w), dtype=np.int64)
        self.values = np.ascontiguousarray(np.asarray(values, dtype=np.int64).reshape(h, w))

    def level(self) -> int:
        return self._level

    def width(self) -> int:
        return self._w

    def height(self) -> int:
        return self._h

    def size(self) -> int:
        return self._w * self._h

    def at(self, ox: int, oy: int) -> int:
        return int(self.values[oy, ox])

    def __eq__(self, other) -> bool:
        return (isinstance(other, CompactGrid) and self._level == other._level and
                np.array_equal(self.values, other.values))


def compact_store(spec: FractalSpec, level: int, embedded: np.ndarray) -> CompactGrid:
    """block_map.cpp:245-262 on the device."""
    n = spec.side_length(level)
    emb = np.ascontiguousarray(embedded, dtype=np.int64)
    if emb.size != n * n:
        raise InvalidArgument(f"compact_store: embedded grid holds {emb.size} cells, expected {n * n}")
    out = CompactGrid(spec, level)
    c = DispatchConfig(spec=spec, r=level, max_cells=max(1 << 24, n * n))
    _check(_lib().nbb_gpu_compact_store(ctypes.byref(c.to_c()), emb.ctypes.data_as(ctypes.c_void_p),
                                        out.values.ctypes.data_as(ctypes.c_void_p)))
    return out


def compact_load(spec: FractalSpec, compact: CompactGrid, empty_value: int = 0) -> np.ndarray:
    """block_map.cpp:264-282 on the device: (n, n) int64, non-members = empty_value."""
    w, h = spec.orthotope_dims(compact.level())
    if (compact.width(), compact.height()) != (w, h):
        raise InvalidArgument(f"compact_load: grid shape does not match spec '{spec.name}' at level "
                              f"{compact.level()}")
    n = spec.side_length(compact.level())
    out = np.empty((n, n), dtype=np.int64)
    c = DispatchConfig(spec=spec, r=compact.level(), max_cells=max(1 << 24, n * n))
    _check(_lib().nbb_gpu_compact_load(ctypes.byref(c.to_c()),
                                       compact.values.ctypes.data_as(ctypes.c_void_p), empty_value,
                                       out.ctypes.data_as(ctypes.c_void_p)))
    return out


def lambda_inverse(spec: FractalSpec, level: int, points) -> np.ndarray:
    """block_map.cpp:113-148 for an (m, 2) array of (x, y) -> (m, 2) array of (ωx, ωy).
    Raises OutOfRange / DomainError for the first offending point, like the reference."""
    xy = np.ascontiguousarray(np.asarray(points, dtype=np.int64).reshape(-1, 2))
    out = np.empty_like(xy)
    c = DispatchConfig(spec=spec)
    _check(_lib().nbb_gpu_lambda_inverse(ctypes.byref(c.to_c()), level,
                                         xy.ctypes.data_as(ctypes.c_void_p), xy.shape[0],
                                         out.ctypes.data_as(ctypes.c_void_p)))
    return out


def write_compact(path: str, spec: FractalSpec, grid: CompactGrid) -> None:
    """NBBC file (block_map.cpp:327-338)."""
    _check(_lib().nbb_gpu_compact_write(str(path).encode(), ctypes.byref(spec.to_c()), grid.level(),
                                        grid.values.ctypes.data_as(ctypes.c_void_p)))


def read_compact(path: str, spec: FractalSpec, max_values: int = 1 << 28) -> CompactGrid:
    """NBBC file (block_map.cpp:340-362)."""
    buf = np.empty(max_values, dtype=np.int64) if max_values <= (1 << 22) else None
    if buf is None:  # size the buffer from the header
        import struct
        with open(path, "rb") as f:
            head = f.read(16)
        lv = struct.unpack("<I", head[12:16])[0] if len(head) == 16 and head[:4] == b"NBBC" else 0
        buf = np.empty(max(1, min(max_values, spec.k ** min(lv, 40))), dtype=np.int64)
    lv = ctypes.c_int32()
    _check(_lib().nbb_gpu_compact_read(str(path).encode(), ctypes.byref(spec.to_c()), ctypes.byref(lv),
                                       buf.ctypes.data_as(ctypes.c_void_p), buf.size))
    w, h = spec.orthotope_dims(lv.value)
    return CompactGrid(spec, lv.value, buf[:w * h].copy())


def device_count() -> int:
    c = ctypes.c_int32()
    _check(_lib().nbb_gpu_device_count(ctypes.byref(c)))
    return c.value


def release() -> None:
    _check(_lib().nbb_gpu_release())
