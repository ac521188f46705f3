"""One nbb_gpu_ca call on pinned host Grids at n = 2^16 (compact state, 1 step), for ncu
(PCIe traffic of the zero-copy member-sector kernels)."""
import ctypes
import os
import sys

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
assert lib.nbb_gpu_ca(ctypes.byref(cc), ctypes.c_void_p(hin.data_ptr()), r, 1, 8, 12,
                      ctypes.c_void_p(hout.data_ptr()), None) == 0
