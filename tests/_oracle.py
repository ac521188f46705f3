"""ctypes bindings for the CHECKERS (test infrastructure only).

  ORC : oracle/_ref/liboracle.so — plain-C restatement (oracle/nbb_oracle.c)
  REF : oracle/_ref/libnbbref.so — the unmodified reference library + our extern "C"
        wrapper (oracle/ref_capi.cpp); built only where /root/reference exists, but the
        .so travels to the GPU box with the snapshot.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_uint16, \
    c_uint64, c_void_p

import numpy as np

from paper_2004_13475_b200 import _abi
from paper_2004_13475_b200.nbb import DispatchConfig, FractalSpec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORC_PATH = os.path.join(ROOT, "oracle", "_ref", "liboracle.so")
REF_PATH = os.path.join(ROOT, "oracle", "_ref", "libnbbref.so")

CP = POINTER(_abi.NbbConfig)
RP = POINTER(_abi.NbbReport)
SP = POINTER(_abi.NbbSpec)
I64P = POINTER(c_int64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(c_void_p)


def fnv1a64(a: np.ndarray) -> str:
    """FNV-1a-64 of the little-endian bytes (SURVEY App. B digest)."""
    lib = orc_lib()
    b = np.ascontiguousarray(a)
    return "%016x" % lib.orc_fnv1a64(_ptr(b), b.nbytes)


_orc = None
_ref = None


def orc_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_PATH):
            raise RuntimeError(f"{ORC_PATH} missing; run __graft_entry__.build()")
        lib = ctypes.CDLL(ORC_PATH)
        sig = {
            "orc_fnv1a64": (c_uint64, [c_void_p, c_size_t]),
            "orc_is_member": (c_int, [SP, c_int, c_int64, c_int64]),
            "orc_gasket_bit_test": (c_int, [c_int, c_int64, c_int64]),
            "orc_lambda_map": (c_int, [SP, c_int, c_int64, c_int64, I64P, I64P]),
            "orc_lambda_inverse": (c_int, [SP, c_int, c_int64, c_int64, I64P, I64P]),
            "orc_lambda_coords": (None, [SP, c_int, c_void_p]),
            "orc_map_thread": (c_int, [SP, c_int, c_int, c_int64, c_int64, c_int64, c_int64, c_int,
                                       I64P, I64P]),
            "orc_random_member_grid": (None, [SP, c_int, c_uint64, c_uint64, c_void_p]),
            "orc_single_write": (None, [SP, c_int, c_void_p]),
            "orc_reduction": (c_int64, [SP, c_int, c_void_p]),
            "orc_ca_step": (None, [SP, c_int, c_void_p, c_void_p, c_uint16, c_uint16]),
            "orc_ca": (None, [SP, c_int, c_void_p, c_int, c_uint16, c_uint16, c_void_p]),
            "orc_random_member_compact": (c_int, [SP, c_int, c_uint64, c_uint64, c_void_p]),
            "orc_ca_compact": (c_int, [SP, c_int, c_void_p, c_int, c_uint16, c_uint16, c_void_p]),
            "orc_ca_compact_check": (c_int64, [SP, c_int, c_void_p, c_void_p, c_void_p, c_int64,
                                               c_uint16, c_uint16]),
            "orc_validate": (c_int, [CP, c_char_p, c_size_t]),
            "orc_plan_report": (c_int, [CP, RP]),
            "orc_launch_block_count": (c_uint64, [CP]),
            "orc_work_quotient": (c_double, [RP, RP, c_int]),
            "orc_csv_row": (None, [RP, c_char_p, c_size_t]),
            "orc_mma_eval": (None, [c_void_p, c_void_p, c_void_p, c_void_p]),
            "orc_encode_variant1": (c_int, [SP, c_int, c_int64, c_int64, c_void_p, c_void_p]),
            "orc_encode_variant2": (c_int, [SP, c_int, c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
            "orc_encode_variant3": (c_int, [SP, c_int, c_int, c_int64, c_int64, c_void_p, c_void_p,
                                            c_void_p, c_void_p, c_void_p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _orc = lib
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref_lib():
    global _ref
    if _ref is None:
        lib = ctypes.CDLL(REF_PATH)
        sig = {
            "ref_last_error": (c_char_p, []),
            "ref_grid_create": (c_void_p, [SP, c_int32]),
            "ref_grid_destroy": (None, [c_void_p]),
            "ref_grid_data": (c_void_p, [c_void_p]),
            "ref_validate": (c_int, [CP]),
            "ref_launch_block_count": (c_int, [CP, POINTER(c_uint64)]),
            "ref_single_write": (c_int, [CP, c_void_p, RP, POINTER(c_double)]),
            "ref_reduction": (c_int, [CP, c_void_p, c_int32, I64P, RP]),
            "ref_reduction_h": (c_int, [CP, c_void_p, I64P, RP, POINTER(c_double)]),
            "ref_ca": (c_int, [CP, c_void_p, c_int32, c_int32, c_uint16, c_uint16, c_void_p, RP,
                               POINTER(c_uint64)]),
            "ref_ca_h": (c_int, [CP, c_void_p, c_int32, c_uint16, c_uint16, c_void_p, RP,
                                 POINTER(c_double)]),
            "ref_random_member_grid": (c_int, [SP, c_int32, c_uint64, c_uint64, c_uint64, c_void_p]),
            "ref_lambda_map": (c_int, [SP, c_int32, c_int64, c_int64, I64P, I64P]),
            "ref_lambda_coords": (c_int, [SP, c_int32, c_void_p]),
            "ref_lambda_inverse": (c_int, [SP, c_int32, c_int64, c_int64, I64P, I64P]),
            "ref_is_member": (c_int, [SP, c_int32, c_int64, c_int64, POINTER(c_int32)]),
            "ref_map_thread": (c_int, [SP, c_int32, c_int32, c_int64, c_int64, c_int64, c_int64,
                                       c_int32, I64P, I64P, POINTER(c_int32)]),
            "ref_mma_variant1": (c_int, [SP, c_int32, c_int64, c_int64, c_void_p]),
            "ref_mma_variant2": (c_int, [SP, c_int32, c_void_p, c_int32, c_void_p, c_void_p]),
            "ref_mma_variant3": (c_int, [SP, c_int32, c_int32, c_int64, c_int64, c_void_p, c_void_p]),
            "ref_work_quotient": (c_int, [RP, RP, c_int32, POINTER(c_double)]),
            "ref_csv_row": (c_int, [RP, c_char_p, c_size_t]),
            "ref_csv_header": (c_char_p, []),
            "ref_compact_store": (c_int, [SP, c_int32, c_void_p, c_void_p]),
            "ref_format_double": (c_int, [c_double, c_char_p, c_size_t]),
            "ref_write_compact": (c_int, [SP, c_int32, c_void_p, c_char_p]),
            "ref_read_compact": (c_int, [SP, c_char_p, POINTER(c_int32), c_void_p, c_uint64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _ref = lib
    return _ref


GASKET = FractalSpec.sierpinski()


# ---- oracle conveniences ----------------------------------------------------------
def orc_random_member_grid(r: int, seed: int, modulus: int, spec: FractalSpec = GASKET) -> np.ndarray:
    n = spec.side_length(r)
    out = np.zeros((n, n), dtype=np.int64)
    orc_lib().orc_random_member_grid(ctypes.byref(spec.to_c()), r, seed, modulus, _ptr(out))
    return out


def orc_single_write(r: int, spec: FractalSpec = GASKET) -> np.ndarray:
    n = spec.side_length(r)
    out = np.zeros((n, n), dtype=np.int64)
    orc_lib().orc_single_write(ctypes.byref(spec.to_c()), r, _ptr(out))
    return out


def orc_reduction(r: int, grid: np.ndarray, spec: FractalSpec = GASKET) -> int:
    g = np.ascontiguousarray(grid, dtype=np.int64)
    return int(orc_lib().orc_reduction(ctypes.byref(spec.to_c()), r, _ptr(g)))


def orc_ca(r: int, grid: np.ndarray, steps: int, birth: int = 8, survive: int = 12,
           spec: FractalSpec = GASKET) -> np.ndarray:
    g = np.ascontiguousarray(grid, dtype=np.int64)
    out = np.empty_like(g)
    orc_lib().orc_ca(ctypes.byref(spec.to_c()), r, _ptr(g), steps, birth, survive, _ptr(out))
    return out


def orc_ca_compact_check(r: int, src: np.ndarray, dst: np.ndarray, offsets: np.ndarray,
                         birth: int = 8, survive: int = 12, spec: FractalSpec = GASKET) -> int:
    """Mismatching sampled offsets of one compact-state CA step src -> dst (oracle rule)."""
    src = np.ascontiguousarray(src, dtype=np.int64).ravel()
    dst = np.ascontiguousarray(dst, dtype=np.int64).ravel()
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    return int(orc_lib().orc_ca_compact_check(ctypes.byref(spec.to_c()), r, _ptr(src), _ptr(dst),
                                              _ptr(offsets), offsets.size, birth, survive))


def orc_random_member_compact(r: int, seed: int, modulus: int, spec: FractalSpec = GASKET) -> np.ndarray:
    """random_member_grid(spec, r, seed, modulus) in compact (λ-ordered) layout, O(3^r)."""
    w, h = 3 ** ((r + 1) // 2), 3 ** (r // 2)
    out = np.zeros(w * h, dtype=np.int64)
    rc = orc_lib().orc_random_member_compact(ctypes.byref(spec.to_c()), r, seed, modulus, _ptr(out))
    if rc:
        raise RuntimeError(f"orc_random_member_compact: status {rc}")
    return out


def orc_ca_compact(r: int, src: np.ndarray, steps: int, birth: int = 8, survive: int = 12,
                   spec: FractalSpec = GASKET) -> np.ndarray:
    """run_ca over a compact state: `steps` steps, compact values out (every cell, any r <= 18)."""
    src = np.ascontiguousarray(src, dtype=np.int64).ravel()
    out = np.empty_like(src)
    rc = orc_lib().orc_ca_compact(ctypes.byref(spec.to_c()), r, _ptr(src), steps, birth, survive, _ptr(out))
    if rc:
        raise RuntimeError(f"orc_ca_compact: status {rc}")
    return out


def orc_lambda_coords(level: int, spec: FractalSpec = GASKET) -> np.ndarray:
    w, h = spec.orthotope_dims(level)
    out = np.empty((w * h, 2), dtype=np.int64)
    orc_lib().orc_lambda_coords(ctypes.byref(spec.to_c()), level, _ptr(out))
    return out


def orc_plan_report(cfg: DispatchConfig):
    rep = _abi.NbbReport()
    rc = orc_lib().orc_plan_report(ctypes.byref(cfg.to_c()), ctypes.byref(rep))
    return rc, rep


def orc_validate(cfg: DispatchConfig):
    buf = ctypes.create_string_buffer(256)
    rc = orc_lib().orc_validate(ctypes.byref(cfg.to_c()), buf, 256)
    return rc, buf.value.decode()


def orc_csv_row(rep) -> str:
    buf = ctypes.create_string_buffer(512)
    orc_lib().orc_csv_row(ctypes.byref(rep), buf, 512)
    return buf.value.decode()


# ---- reference conveniences ---------------------------------------------------------
def _ref_check(rc: int):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {ref_lib().ref_last_error().decode()}")


def ref_random_member_grid(r: int, seed: int, modulus: int, spec: FractalSpec = GASKET) -> np.ndarray:
    n = spec.side_length(r)
    out = np.zeros((n, n), dtype=np.int64)
    _ref_check(ref_lib().ref_random_member_grid(ctypes.byref(spec.to_c()), r, seed, modulus,
                                                max(1 << 24, n * n), _ptr(out)))
    return out


def ref_single_write(cfg: DispatchConfig):
    n = cfg.spec.side_length(cfg.r)
    out = np.zeros((n, n), dtype=np.int64)
    rep = _abi.NbbReport()
    rc = ref_lib().ref_single_write(ctypes.byref(cfg.to_c()), _ptr(out), ctypes.byref(rep), None)
    return rc, out, rep


def ref_reduction(cfg: DispatchConfig, grid: np.ndarray, level: int):
    v = c_int64()
    rep = _abi.NbbReport()
    g = np.ascontiguousarray(grid, dtype=np.int64)
    rc = ref_lib().ref_reduction(ctypes.byref(cfg.to_c()), _ptr(g), level, ctypes.byref(v),
                                 ctypes.byref(rep))
    return rc, v.value, rep


def ref_ca(cfg: DispatchConfig, grid: np.ndarray, steps: int, birth: int = 8, survive: int = 12):
    g = np.ascontiguousarray(grid, dtype=np.int64)
    out = np.empty_like(g)
    reps = (_abi.NbbReport * max(steps, 1))()
    gen = c_uint64()
    rc = ref_lib().ref_ca(ctypes.byref(cfg.to_c()), _ptr(g), cfg.r, steps, birth, survive,
                          _ptr(out), reps, ctypes.byref(gen))
    return rc, out, [reps[i] for i in range(steps)]


def ref_lambda_coords(level: int, spec: FractalSpec = GASKET) -> np.ndarray:
    w, h = spec.orthotope_dims(level)
    out = np.empty((w * h, 2), dtype=np.int64)
    _ref_check(ref_lib().ref_lambda_coords(ctypes.byref(spec.to_c()), level, _ptr(out)))
    return out


def ref_validate(cfg: DispatchConfig):
    rc = ref_lib().ref_validate(ctypes.byref(cfg.to_c()))
    return rc, (ref_lib().ref_last_error().decode() if rc else "")


def ref_csv_row(rep) -> str:
    buf = ctypes.create_string_buffer(512)
    _ref_check(ref_lib().ref_csv_row(ctypes.byref(rep), buf, 512))
    return buf.value.decode()
