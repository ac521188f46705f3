"""Wall time of nbb_gpu_ca on pinned host buffers at n = 2^16 (compact state, FLAG_OUT_ZEROED):
steps = 1 (transfer-dominated) and steps = 200."""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import _abi, nbb  # noqa: E402

r, n = 16, 1 << 16
spec = nbb.FractalSpec.sierpinski()
lib = _abi.load()
hin = torch.empty((n, n), dtype=torch.int64, pin_memory=True)
hout = torch.zeros((n, n), dtype=torch.int64).pin_memory()
lib.nbb_gpu_random_member_grid(ctypes.byref(spec.to_c()), r, 17, 2, n * n, ctypes.c_void_p(hin.data_ptr()))
cc = nbb.DispatchConfig(r=r, rho=32, max_cells=n * n,
                        flags=_abi.FLAG_OUT_ZEROED | _abi.FLAG_COMPACT_STATE).to_c()


def call(steps):
    t0 = time.perf_counter()
    rc = lib.nbb_gpu_ca(ctypes.byref(cc), ctypes.c_void_p(hin.data_ptr()), r, steps, 8, 12,
                        ctypes.c_void_p(hout.data_ptr()), None)
    assert rc == 0, lib.nbb_gpu_last_error()
    return time.perf_counter() - t0


call(1)
res = {
       "one_step_s": min(call(1) for _ in range(5)), "k200_s": min(call(200) for _ in range(3))}
res["cells_per_s_k200"] = 3 ** r * 200 / res["k200_s"]
print(json.dumps(res))
