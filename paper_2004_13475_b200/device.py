"""Device-resident entry points (the `*_dev` half of include/nbb_gpu.h).

Pointers are raw device addresses (e.g. ``tensor.data_ptr()``) and ``stream`` is a
cudaStream_t handle as an int (e.g. ``torch.cuda.current_stream().cuda_stream``),
so a caller can keep grids resident in HBM and time launches with CUDA events on
the same stream. No host synchronisation happens inside these calls unless
``config.timing`` is set.
"""
from __future__ import annotations

import ctypes

from . import _abi
from .nbb import CaRule, DispatchConfig, WorkReport, _check, _lib


def _vp(x: int):
    return ctypes.c_void_p(int(x))


def single_write_dev(config: DispatchConfig, d_grid: int, stream: int = 0) -> WorkReport:
    rep = _abi.NbbReport()
    _check(_lib().nbb_gpu_single_write_dev(ctypes.byref(config.to_c()), _vp(d_grid), _vp(stream),
                                           ctypes.byref(rep)))
    return WorkReport.from_c(rep)


def reduction_dev(config: DispatchConfig, d_grid: int, d_value: int, stream: int = 0) -> WorkReport:
    rep = _abi.NbbReport()
    _check(_lib().nbb_gpu_reduction_dev(ctypes.byref(config.to_c()), _vp(d_grid), _vp(d_value),
                                        _vp(stream), ctypes.byref(rep)))
    return WorkReport.from_c(rep)


def ca_step_dev(config: DispatchConfig, d_src: int, d_dst: int, rule: CaRule = CaRule(),
                stream: int = 0) -> WorkReport:
    rep = _abi.NbbReport()
    _check(_lib().nbb_gpu_ca_step_dev(ctypes.byref(config.to_c()), _vp(d_src), _vp(d_dst),
                                      rule.birth, rule.survive, _vp(stream), ctypes.byref(rep)))
    return WorkReport.from_c(rep)


def ca_run_dev(config: DispatchConfig, d_a: int, d_b: int, steps: int, rule: CaRule = CaRule(),
               stream: int = 0) -> "_abi.NbbPassStats":
    """`steps` steps on an embedded device grid (result in d_a for even steps, else d_b); the gasket's
    int64 grid runs temporally blocked through the compact state (nbb_gpu_ca_run_dev)."""
    st = _abi.NbbPassStats()
    _check(_lib().nbb_gpu_ca_run_dev(ctypes.byref(config.to_c()), _vp(d_a), _vp(d_b), steps, rule.birth,
                                     rule.survive, _vp(stream), ctypes.byref(st)))
    return st


def sanitize_dev(config: DispatchConfig, d_grid: int, stream: int = 0) -> None:
    _check(_lib().nbb_gpu_sanitize_dev(ctypes.byref(config.to_c()), _vp(d_grid), _vp(stream)))


def pack_alive_dev(config: DispatchConfig, d_grid64: int, d_grid8: int, stream: int = 0) -> None:
    _check(_lib().nbb_gpu_pack_alive_dev(ctypes.byref(config.to_c()), _vp(d_grid64), _vp(d_grid8),
                                         _vp(stream)))


def unpack_alive_dev(config: DispatchConfig, d_grid8: int, d_grid64: int, stream: int = 0) -> None:
    _check(_lib().nbb_gpu_unpack_alive_dev(ctypes.byref(config.to_c()), _vp(d_grid8),
                                           _vp(d_grid64), _vp(stream)))


def scatter_members_dev(config: DispatchConfig, d_values: int, d_grid: int, stream: int = 0) -> None:
    _check(_lib().nbb_gpu_scatter_members_dev(ctypes.byref(config.to_c()), _vp(d_values),
                                              _vp(d_grid), _vp(stream)))


def compact_store_dev(config: DispatchConfig, d_embedded: int, d_compact: int, stream: int = 0) -> None:
    _check(_lib().nbb_gpu_compact_store_dev(ctypes.byref(config.to_c()), _vp(d_embedded),
                                            _vp(d_compact), _vp(stream)))


def compact_load_dev(config: DispatchConfig, d_compact: int, d_embedded: int, empty_value: int = 0,
                     stream: int = 0) -> None:
    _check(_lib().nbb_gpu_compact_load_dev(ctypes.byref(config.to_c()), _vp(d_compact), empty_value,
                                           _vp(d_embedded), _vp(stream)))


def ca_compact_step_dev(config: DispatchConfig, d_src: int, d_dst: int, rule: CaRule = CaRule(),
                        stream: int = 0) -> WorkReport:
    rep = _abi.NbbReport()
    _check(_lib().nbb_gpu_ca_compact_step_dev(ctypes.byref(config.to_c()), _vp(d_src), _vp(d_dst),
                                              rule.birth, rule.survive, _vp(stream), ctypes.byref(rep)))
    return WorkReport.from_c(rep)


def ca_compact_run_dev(config: DispatchConfig, d_a: int, d_b: int, steps: int, rule: CaRule = CaRule(),
                       stream: int = 0) -> None:
    """`steps` steps ping-ponging d_a <-> d_b, issued by the library (result in d_a if steps
    is even, else d_b)."""
    _check(_lib().nbb_gpu_ca_compact_run_dev(ctypes.byref(config.to_c()), _vp(d_a), _vp(d_b), steps,
                                             rule.birth, rule.survive, _vp(stream)))


def ca_compact_passes_dev(config: DispatchConfig, d_a: int, d_b: int, steps: int, rule: CaRule = CaRule(),
                          stream: int = 0, parity: bool = False) -> "_abi.NbbPassStats":
    """`steps` steps in passes of up to config.pass_steps steps (default 8); without `parity`
    the fewest passes, the result in d_b iff the returned stats.result_in_b."""
    st = _abi.NbbPassStats()
    _check(_lib().nbb_gpu_ca_compact_passes_dev(ctypes.byref(config.to_c()), _vp(d_a), _vp(d_b), steps,
                                                rule.birth, rule.survive, 1 if parity else 0, _vp(stream),
                                                ctypes.byref(st)))
    return st


def pass_plan(config: DispatchConfig, steps: int, parity: bool = False) -> "_abi.NbbPassStats":
    """Host only: the passes a compact CA run of `steps` steps issues."""
    st = _abi.NbbPassStats()
    _check(_lib().nbb_gpu_pass_plan(ctypes.byref(config.to_c()), steps, 1 if parity else 0, ctypes.byref(st)))
    return st


def reduction_compact_dev(config: DispatchConfig, d_compact: int, d_value: int, stream: int = 0) -> WorkReport:
    rep = _abi.NbbReport()
    _check(_lib().nbb_gpu_reduction_compact_dev(ctypes.byref(config.to_c()), _vp(d_compact),
                                                _vp(d_value), _vp(stream), ctypes.byref(rep)))
    return WorkReport.from_c(rep)


def single_write_compact_dev(config: DispatchConfig, d_compact: int, stream: int = 0) -> WorkReport:
    rep = _abi.NbbReport()
    _check(_lib().nbb_gpu_single_write_compact_dev(ctypes.byref(config.to_c()), _vp(d_compact),
                                                   _vp(stream), ctypes.byref(rep)))
    return WorkReport.from_c(rep)


def lambda_coords_dev(config: DispatchConfig, level: int, d_xy: int, coord_bytes: int = 4,
                      stream: int = 0) -> None:
    _check(_lib().nbb_gpu_lambda_coords_dev(ctypes.byref(config.to_c()), level, _vp(d_xy),
                                            coord_bytes, _vp(stream)))
