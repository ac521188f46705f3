"""ctypes view of the C ABI declared in include/nbb_gpu.h.

The product library is ``paper_2004_13475_b200/libnbbgpu.so`` (built in-tree by
``__graft_entry__.build()``). Loading fails loudly when it is missing: there is
no Python or CPU fallback for any compute entry point.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char, c_char_p, c_double, c_int, c_int32, c_int64,
                    c_size_t, c_uint16, c_uint64, c_void_p)

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NBB_GPU_LIB") or os.path.join(PKG_DIR, "libnbbgpu.so")  # env: tuning builds

MAX_REPLICAS = 9

# status codes (nbb_status)
OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_OUT_OF_RANGE = 2
ERR_RESOURCE = 3
ERR_CUDA = 4
ERR_NCCL = 5
ERR_DOMAIN = 6
ERR_OVERFLOW = 7
ERR_RUNTIME = 8

MODE_BB, MODE_LAMBDA = 0, 1
STRATEGY_UNROLL, STRATEGY_LUT, STRATEGY_SUBBOX = 0, 1, 2
BACKEND_DIRECT, BACKEND_MMA1, BACKEND_MMA2, BACKEND_MMA3 = 0, 1, 2, 3
KERNEL_AUTO, KERNEL_PERCELL, KERNEL_TILE = 0, 1, 2


class NbbSpec(Structure):
    _fields_ = [
        ("name", c_char * 32),
        ("k", c_int32),
        ("s", c_int32),
        ("offset_x", c_int32 * MAX_REPLICAS),
        ("offset_y", c_int32 * MAX_REPLICAS),
    ]


class NbbConfig(Structure):
    _fields_ = [
        ("spec", NbbSpec),
        ("r", c_int32),
        ("rho", c_int32),
        ("mode", c_int32),
        ("strategy", c_int32),
        ("backend", c_int32),
        ("workers", c_int32),
        ("timing", c_int32),
        ("cell_width", c_int32),
        ("kernel", c_int32),
        ("device", c_int32),
        ("max_cells", c_uint64),
        ("shard_begin", c_uint64),
        ("shard_count", c_uint64),
        ("flags", ctypes.c_uint32),
        ("pass_steps", ctypes.c_uint32),
    ]


FLAG_OUT_ZEROED = 1
FLAG_COMPACT_STATE = 2
FLAG_SINGLE_STEP = 4
FLAG_EMBEDDED_STATE = 8


class NbbReport(Structure):
    _fields_ = [
        ("spec_name", c_char * 32),
        ("r", c_int32),
        ("rho", c_int32),
        ("mode", c_int32),
        ("strategy", c_int32),
        ("backend", c_int32),
        ("map_levels", c_int32),
        ("blocks_launched", c_uint64),
        ("threads_launched", c_uint64),
        ("threads_active", c_uint64),
        ("threads_wasted", c_uint64),
        ("map_ops", c_uint64),
        ("micros", c_uint64),
    ]


class NbbPassStats(Structure):
    """nbb_pass_stats (nbb_gpu.h): the passes a compact CA run issued."""
    _fields_ = [
        ("passes", c_int32),
        ("by_steps", c_int32 * 13),
        ("result_in_b", c_int32),
    ]


class NbbP2P(Structure):
    """nbb_p2p (nbb_gpu.h): one rank's view of the multi-GPU compact CA."""
    _fields_ = [
        ("world", c_int32),
        ("rank", c_int32),
        ("d_buf", c_void_p * 2),
        ("d_peer_buf", c_void_p * 2),
        ("reserved", c_void_p),
        ("d_sync", c_void_p),
        ("d_peer_flag", c_void_p),
        ("timeout_ms", ctypes.c_uint32),
    ]


CP = POINTER(NbbConfig)
RP = POINTER(NbbReport)
SP = POINTER(NbbSpec)
I64P = POINTER(c_int64)

# name -> (restype, argtypes); every symbol include/nbb_gpu.h declares.
SIGNATURES = {
    "nbb_gpu_abi_version": (c_int, []),
    "nbb_gpu_last_error": (c_char_p, []),
    "nbb_config_init": (None, [CP]),
    "nbb_spec_sierpinski": (None, [SP]),
    "nbb_spec_vicsek": (None, [SP]),
    "nbb_spec_carpet": (None, [SP]),
    "nbb_gpu_device_count": (c_int, [POINTER(c_int32)]),
    "nbb_gpu_validate": (c_int, [CP]),
    "nbb_gpu_launch_block_count": (c_int, [CP, POINTER(c_uint64)]),
    "nbb_gpu_plan_report": (c_int, [CP, RP]),
    "nbb_gpu_work_quotient": (c_int, [RP, RP, c_int32, POINTER(c_double)]),
    "nbb_gpu_csv_header": (c_char_p, []),
    "nbb_gpu_report_csv_row": (c_int, [RP, c_char_p, c_size_t]),
    "nbb_gpu_random_member_grid": (c_int, [SP, c_int32, c_uint64, c_uint64, c_uint64, c_void_p]),
    "nbb_gpu_random_member_values": (c_int, [SP, c_int32, c_uint64, c_uint64, c_void_p]),
    "nbb_gpu_single_write": (c_int, [CP, c_void_p, RP]),
    "nbb_gpu_reduction": (c_int, [CP, c_void_p, c_int32, I64P, RP]),
    "nbb_gpu_ca": (c_int, [CP, c_void_p, c_int32, c_int32, c_uint16, c_uint16, c_void_p, RP]),
    "nbb_gpu_lambda_coords": (c_int, [CP, c_int32, c_void_p]),
    "nbb_gpu_ca_multi": (c_int, [CP, POINTER(c_int32), c_int32, c_void_p, c_int32, c_int32, c_uint16, c_uint16,
                                 c_void_p, RP]),
    "nbb_gpu_reduction_multi": (c_int, [CP, POINTER(c_int32), c_int32, c_void_p, c_int32, I64P, RP]),
    "nbb_gpu_single_write_dev": (c_int, [CP, c_void_p, c_void_p, RP]),
    "nbb_gpu_reduction_dev": (c_int, [CP, c_void_p, c_void_p, c_void_p, RP]),
    "nbb_gpu_ca_step_dev": (c_int, [CP, c_void_p, c_void_p, c_uint16, c_uint16, c_void_p, RP]),
    "nbb_gpu_sanitize_dev": (c_int, [CP, c_void_p, c_void_p]),
    "nbb_gpu_ca_run_dev": (c_int, [CP, c_void_p, c_void_p, c_int32, c_uint16, c_uint16, c_void_p,
                                   POINTER(NbbPassStats)]),
    "nbb_gpu_pack_alive_dev": (c_int, [CP, c_void_p, c_void_p, c_void_p]),
    "nbb_gpu_unpack_alive_dev": (c_int, [CP, c_void_p, c_void_p, c_void_p]),
    "nbb_gpu_scatter_members_dev": (c_int, [CP, c_void_p, c_void_p, c_void_p]),
    "nbb_gpu_lambda_coords_dev": (c_int, [CP, c_int32, c_void_p, c_int32, c_void_p]),
    "nbb_gpu_gather_cells_dev": (c_int, [CP, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "nbb_gpu_scatter_cells_dev": (c_int, [CP, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "nbb_gpu_release": (c_int, []),
    "nbb_gpu_compact_store": (c_int, [CP, c_void_p, c_void_p]),
    "nbb_gpu_compact_load": (c_int, [CP, c_void_p, c_int64, c_void_p]),
    "nbb_gpu_compact_store_dev": (c_int, [CP, c_void_p, c_void_p, c_void_p]),
    "nbb_gpu_compact_load_dev": (c_int, [CP, c_void_p, c_int64, c_void_p, c_void_p]),
    "nbb_gpu_lambda_inverse": (c_int, [CP, c_int32, c_void_p, c_uint64, c_void_p]),
    "nbb_gpu_compact_write": (c_int, [ctypes.c_char_p, SP, c_int32, c_void_p]),
    "nbb_gpu_compact_read": (c_int, [ctypes.c_char_p, SP, POINTER(c_int32), c_void_p, c_uint64]),
    "nbb_gpu_ca_compact_step_dev": (c_int, [CP, c_void_p, c_void_p, c_uint16, c_uint16, c_void_p, RP]),
    "nbb_gpu_reduction_compact_dev": (c_int, [CP, c_void_p, c_void_p, c_void_p, RP]),
    "nbb_gpu_single_write_compact_dev": (c_int, [CP, c_void_p, c_void_p, RP]),
    "nbb_gpu_ca_compact_run_dev": (c_int, [CP, c_void_p, c_void_p, c_int32, c_uint16, c_uint16, c_void_p]),
    "nbb_gpu_ca_compact_passes_dev": (c_int, [CP, c_void_p, c_void_p, c_int32, c_uint16, c_uint16, c_int32,
                                              c_void_p, POINTER(NbbPassStats)]),
    "nbb_gpu_pass_plan": (c_int, [CP, c_int32, c_int32, POINTER(NbbPassStats)]),
    "nbb_gpu_ca_compact_p2p_dev": (c_int, [CP, ctypes.c_int64, c_int32, c_uint16, c_uint16,
                                           POINTER(NbbP2P), c_void_p]),
    "nbb_gpu_ca_compact_p2p_passes_dev": (c_int, [CP, ctypes.c_int64, c_int32, c_uint16, c_uint16,
                                                  POINTER(NbbP2P), c_void_p]),
    "nbb_gpu_comm_unique_id": (c_int, [POINTER(ctypes.c_uint8)]),
    "nbb_gpu_comm_init": (c_int, [POINTER(ctypes.c_uint8), c_int32, c_int32, c_int32, POINTER(c_void_p)]),
    "nbb_gpu_comm_destroy": (c_int, [c_void_p]),
    "nbb_gpu_ca_compact_comm_dev": (c_int, [CP, c_void_p, c_void_p, c_void_p, c_int32, c_uint16, c_uint16,
                                            c_void_p, POINTER(NbbPassStats)]),
    "nbb_gpu_reduction_compact_comm_dev": (c_int, [CP, c_void_p, c_void_p, c_void_p, c_void_p]),
    "nbb_gpu_halo_exchange_counts": (c_int, [CP, c_int32, c_int32, c_int32, POINTER(c_uint64), POINTER(c_uint64)]),
    "nbb_gpu_halo_exchange_lists": (c_int, [CP, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p]),
    "nbb_gpu_p2p_check": (c_int, [POINTER(NbbP2P), c_void_p]),
    "nbb_gpu_malloc": (c_int, [c_int32, c_uint64, POINTER(c_void_p)]),
    "nbb_gpu_free": (c_int, [c_int32, c_void_p]),
    "nbb_gpu_ipc_handle": (c_int, [c_int32, c_void_p, POINTER(ctypes.c_uint8)]),
    "nbb_gpu_ipc_open": (c_int, [c_int32, POINTER(ctypes.c_uint8), POINTER(c_void_p)]),
    "nbb_gpu_ipc_close": (c_int, [c_int32, c_void_p]),
}

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the in-tree product library (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the GPU path)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
