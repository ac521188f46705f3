"""Per-cell λ launch (the paper's kernels) at n = 2^16, ρ = 16, SW: direct vs the MMA backends."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import device as dev  # noqa: E402
from paper_2004_13475_b200 import nbb  # noqa: E402

n = 1 << 16
s = torch.cuda.current_stream().cuda_stream
b = torch.zeros((n, n), dtype=torch.int64, device="cuda")
res = {}
for name, be in (("direct", nbb.LambdaBackend.Direct), ("mma1", nbb.LambdaBackend.MmaV1),
                 ("mma2", nbb.LambdaBackend.MmaV2), ("mma3", nbb.LambdaBackend.MmaV3)):
    c = nbb.DispatchConfig(r=16, rho=16, kernel=nbb.KernelFamily.PerCell, backend=be, max_cells=n * n)
    for _ in range(2):
        dev.single_write_dev(c, b.data_ptr(), s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dev.single_write_dev(c, b.data_ptr(), s)
    e1.record()
    e1.synchronize()
    res[name] = e0.elapsed_time(e1) / 10
print(json.dumps(res))
