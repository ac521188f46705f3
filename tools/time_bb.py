"""BB vs λ launch shapes on the embedded int64 grid at n = 2^16 (CA, SW, RD), CUDA events."""
import json
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
c = nbb.DispatchConfig(r=r, rho=32, max_cells=n * n)
dev.scatter_members_dev(c, vals.data_ptr(), a.data_ptr(), s)
b = torch.zeros_like(a)
out = torch.zeros(1, dtype=torch.int64, device="cuda")


def cfg(**kw):
    x = nbb.DispatchConfig(r=r, rho=32, max_cells=n * n)
    for k, v in kw.items():
        setattr(x, k, v)
    return x


def timed(fn, K=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / K


BB = nbb.MapMode.BoundingBox
res = {}
for name, c in {"ca_lambda_tile": cfg(), "ca_bb_tile": cfg(mode=BB), "ca_bb_tile_rho16": cfg(mode=BB, rho=16)}.items():
    res[name] = timed(lambda: dev.ca_step_dev(c, a.data_ptr(), b.data_ptr(), nbb.CaRule(), s))
for name, c in {"sw_lambda_tile": cfg(), "sw_bb_tile": cfg(mode=BB)}.items():
    res[name] = timed(lambda: dev.single_write_dev(c, b.data_ptr(), s))
for name, c in {"rd_lambda_tile": cfg(), "rd_bb_tile": cfg(mode=BB)}.items():
    res[name] = timed(lambda: dev.reduction_dev(c, a.data_ptr(), out.data_ptr(), s))
# the two launches give the same grid
dev.ca_step_dev(cfg(), a.data_ptr(), b.data_ptr(), nbb.CaRule(), s)
ref = b.clone()
b.zero_()
dev.ca_step_dev(cfg(mode=BB), a.data_ptr(), b.data_ptr(), nbb.CaRule(), s)
res["bb_equals_lambda"] = bool(torch.equal(ref, b))
print(json.dumps(res))
