"""A few CA steps of each state layout at n = 2^16 (λ, ρ = 32), for ncu captures:
    ncu --set full -k regex:<kernel> -c 2 -o prof python tools/profile_ca.py [bits|i64|u8|bb]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import device as dev  # noqa: E402
from paper_2004_13475_b200 import nbb  # noqa: E402

which = sys.argv[1:] or ["bits", "i64", "u8"]
r, n = 16, 1 << 16
s = torch.cuda.current_stream().cuda_stream
spec = nbb.FractalSpec.sierpinski()
a = torch.zeros((n, n), dtype=torch.int64, device="cuda")
vals = torch.from_numpy(nbb.random_member_values(spec, r, 17, 2)).cuda()
c64 = nbb.DispatchConfig(r=r, rho=32, max_cells=n * n)
dev.scatter_members_dev(c64, vals.data_ptr(), a.data_ptr(), s)
del vals
if "bits" in which:
    c = nbb.DispatchConfig(r=r, rho=32, max_cells=n * n, cell_width=0)
    w1 = torch.zeros((n, n // 32), dtype=torch.int32, device="cuda")
    w2 = torch.zeros_like(w1)
    dev.pack_alive_dev(c, a.data_ptr(), w1.data_ptr(), s)
    for i in range(4):
        dev.ca_step_dev(c, (w1 if i % 2 == 0 else w2).data_ptr(), (w2 if i % 2 == 0 else w1).data_ptr(),
                        nbb.CaRule(), s)
if "u8" in which:
    c = nbb.DispatchConfig(r=r, rho=32, max_cells=n * n, cell_width=1)
    a8 = torch.zeros((n, n), dtype=torch.uint8, device="cuda")
    b8 = torch.zeros_like(a8)
    dev.pack_alive_dev(c, a.data_ptr(), a8.data_ptr(), s)
    for i in range(4):
        dev.ca_step_dev(c, (a8 if i % 2 == 0 else b8).data_ptr(), (b8 if i % 2 == 0 else a8).data_ptr(),
                        nbb.CaRule(), s)
if "i64" in which or "bb" in which:
    b = torch.zeros_like(a)
    c = c64 if "i64" in which else nbb.DispatchConfig(r=r, rho=32, max_cells=n * n,
                                                      mode=nbb.MapMode.BoundingBox)
    for i in range(4):
        dev.ca_step_dev(c, (a if i % 2 == 0 else b).data_ptr(), (b if i % 2 == 0 else a).data_ptr(),
                        nbb.CaRule(), s)
torch.cuda.synchronize()
