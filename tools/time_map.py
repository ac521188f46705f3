"""C4 timing: the λ map over whole orthotopes, scalar K0 (int32 pairs), CUDA events."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import device as dev  # noqa: E402
from paper_2004_13475_b200 import nbb  # noqa: E402

s = torch.cuda.current_stream().cuda_stream
xy = torch.empty(3 ** 17 * 2, dtype=torch.int32, device="cuda")
res = {}
for lvl in (14, 16, 17):
    c = nbb.DispatchConfig(r=16, rho=32)
    for _ in range(3):
        dev.lambda_coords_dev(c, lvl, xy.data_ptr(), 4, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        dev.lambda_coords_dev(c, lvl, xy.data_ptr(), 4, s)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 50
    res[lvl] = {"ms": ms, "GBps": 3 ** lvl * 8 / ms / 1e6}
print(json.dumps(res))
