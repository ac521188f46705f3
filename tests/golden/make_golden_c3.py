"""Generate tests/golden/c3_r16.json by running the UNMODIFIED reference at the headline size.

C3 (BASELINE configs[2]): the gasket at n = 2^16, initial = random_member_grid(gasket, 16,
seed 17, modulus 2), rule B3/S23 (plus B25/S34 for the generic-rule kernels: member cells have 2-5 member
neighbours, so only the rule bits of counts 0..5 can matter). The reference
(oracle/_ref/libnbbref.so, built from /root/reference/proj/src by oracle/Makefile; the .so
travels to the GPU box) needs ~140 GB of host RAM here (two 32 GiB Grids inside run_ca, its
4 GiB MemberMask, our input / output Grids), so this runs on the GPU box's host, not in the
CPU container (62 GB):

    gpurun -- python tests/golden/make_golden_c3.py gpurun_out/c3_r16.json

Each trajectory is run_ca(cfg, grid, Δ) chained from the previous output (run_ca is a pure
function of the state, dispatch.cpp:517-557, so run_ca(run_ca(g, a), b) == run_ca(g, a + b)).
Recorded per step count: the population and the FNV-1a-64 of the state in COMPACT order
(value(ω) = grid[λ(ω)], i.e. the reference's compact_store, block_map.cpp:245-263, of its
output Grid) — the form the GPU's compact state and the oracle's orc_ca_compact produce.
Nothing from the product library (libnbbgpu.so) is loaded.
"""
from __future__ import annotations

import ctypes
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from _oracle import GASKET, fnv1a64, ref_lambda_coords, ref_lib  # noqa: E402
from paper_2004_13475_b200 import _abi  # noqa: E402  (ctypes struct layouts only)
from paper_2004_13475_b200.nbb import DispatchConfig  # noqa: E402

R, SEED = int(os.environ.get("C3_LEVEL", "16")), 17
TRAJECTORIES = {"B3/S23": ((1 << 3, (1 << 2) | (1 << 3)), (1, 2, 3, 4, 5, 8, 20)),
                "B25/S34": (((1 << 2) | (1 << 5), (1 << 3) | (1 << 4)), (1, 2, 4))}


def mem_gb() -> float:
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith("MemAvailable"):
                return int(line.split()[1]) / 2 ** 20
    return -1.0


def main(out_path: str) -> None:
    ref = ref_lib()
    n = 1 << R
    spec = GASKET.to_c()
    t0 = time.time()
    xy = ref_lambda_coords(R)                          # compact offset -> (x, y), the reference's λ
    flat = xy[:, 1] * n + xy[:, 0]
    del xy
    cores = os.cpu_count() or 1
    cfg = DispatchConfig(r=R, rho=32, workers=cores, timing=True, max_cells=n * n).to_c()

    def grid_view(h):
        return np.ctypeslib.as_array(ctypes.cast(ref.ref_grid_data(h), ctypes.POINTER(ctypes.c_int64)),
                                     shape=(n * n,))

    out = {"r": R, "seed": SEED, "modulus": 2, "layout": "compact (value(omega) = grid[lambda(omega)])",
           "digest": "FNV-1a-64 over the little-endian int64 compact values",
           "generator": "tests/golden/make_golden_c3.py (unmodified reference via oracle/_ref/libnbbref.so)",
           "host": {"cores": cores, "mem_available_gb_at_start": round(mem_gb(), 1)},
           "trajectories": {}}
    for name, ((birth, survive), steps_list) in TRAJECTORIES.items():
        h = ref.ref_grid_create(ctypes.byref(spec), R)
        rc = ref.ref_random_member_grid(ctypes.byref(spec), R, SEED, 2, n * n,
                                        ctypes.c_void_p(ref.ref_grid_data(h)))
        assert rc == 0, ref.ref_last_error()
        c0 = grid_view(h)[flat]
        traj = {"birth": birth, "survive": survive,
                "0": {"population": int(c0.sum()), "fnv": fnv1a64(c0)}}
        done = 0
        for target in steps_list:
            nxt = ref.ref_grid_create(ctypes.byref(spec), R)
            reps = (_abi.NbbReport * (target - done))()
            secs = ctypes.c_double()
            rc = ref.ref_ca_h(ctypes.byref(cfg), h, target - done, birth, survive, nxt, reps,
                              ctypes.byref(secs))
            assert rc == 0, ref.ref_last_error()
            ref.ref_grid_destroy(h)
            h, done = nxt, target
            c = grid_view(h)[flat]
            traj[str(target)] = {"population": int(c.sum()), "fnv": fnv1a64(c),
                                 "call_seconds": round(secs.value, 2)}
            print(name, target, traj[str(target)], f"mem {mem_gb():.0f} GB", flush=True)
        ref.ref_grid_destroy(h)
        out["trajectories"][name] = traj
    out["seconds"] = round(time.time() - t0, 1)
    os.makedirs(os.path.dirname(os.path.abspath(out_path)), exist_ok=True)
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "c3_r16.json"))
