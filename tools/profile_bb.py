"""One BB tile launch each of RD, CA and SW at n = 2^16 (ρ = 32, int64), for ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import device as dev  # noqa: E402
from paper_2004_13475_b200 import nbb  # noqa: E402

r, n = 16, 1 << 16
s = torch.cuda.current_stream().cuda_stream
a = torch.zeros((n, n), dtype=torch.int64, device="cuda")
vals = torch.from_numpy(nbb.random_member_values(nbb.FractalSpec.sierpinski(), r, 17, 2)).cuda()
c = nbb.DispatchConfig(r=r, rho=32, max_cells=n * n, mode=nbb.MapMode.BoundingBox)
dev.scatter_members_dev(c, vals.data_ptr(), a.data_ptr(), s)
b = torch.zeros_like(a)
out = torch.zeros(1, dtype=torch.int64, device="cuda")
dev.reduction_dev(c, a.data_ptr(), out.data_ptr(), s)
dev.ca_step_dev(c, a.data_ptr(), b.data_ptr(), nbb.CaRule(), s)
dev.single_write_dev(c, b.data_ptr(), s)
torch.cuda.synchronize()
