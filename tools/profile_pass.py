"""A few compact CA passes at n = 2^16 for ncu (prints nothing): python tools/profile_pass.py K [BB]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import nbb  # noqa: E402
from paper_2004_13475_b200 import device as dev  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
mode = nbb.MapMode.BoundingBox if len(sys.argv) > 2 and sys.argv[2] == "BB" else nbb.MapMode.Lambda
r = 16
s = torch.cuda.current_stream().cuda_stream
a = torch.randint(0, 2, (3 ** r,), dtype=torch.int64, device="cuda")
b = torch.empty_like(a)
c = nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, pass_steps=K, mode=mode)
dev.ca_compact_passes_dev(c, a.data_ptr(), b.data_ptr(), 3 * K, nbb.CaRule(), s)
torch.cuda.synchronize()
