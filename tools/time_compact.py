"""Time the compact-state (λ-ordered CompactGrid) workloads at n = 2^16."""
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
spec = nbb.FractalSpec.sierpinski()
c = nbb.DispatchConfig(r=r, rho=32, max_cells=n * n)
a = torch.zeros((n, n), dtype=torch.int64, device="cuda")
vals = torch.from_numpy(nbb.random_member_values(spec, r, 17, 2)).cuda()
dev.scatter_members_dev(c, vals.data_ptr(), a.data_ptr(), s)
c1 = torch.empty(3 ** r, dtype=torch.int64, device="cuda")
c2 = torch.empty_like(c1)
dev.compact_store_dev(c, a.data_ptr(), c1.data_ptr(), s)
out = torch.zeros(1, dtype=torch.int64, device="cuda")


def timed(fn, K=100):
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


res = {
    "ca_compact_ms": timed(lambda: dev.ca_compact_step_dev(c, c1.data_ptr(), c2.data_ptr(), nbb.CaRule(), s)),
    "rd_compact_ms": timed(lambda: dev.reduction_compact_dev(c, c1.data_ptr(), out.data_ptr(), s)),
    "sw_compact_ms": timed(lambda: dev.single_write_compact_dev(c, c2.data_ptr(), s)),
    "compact_store_ms": timed(lambda: dev.compact_store_dev(c, a.data_ptr(), c1.data_ptr(), s), 10),
}
back = torch.zeros_like(a)
dev.compact_load_dev(c, c1.data_ptr(), back.data_ptr(), 0, s)
res["codec_roundtrip_exact"] = bool(torch.equal(back, a))
ref = torch.zeros_like(a)
dev.ca_step_dev(c, a.data_ptr(), ref.data_ptr(), nbb.CaRule(), s)
dev.ca_compact_step_dev(c, c1.data_ptr(), c2.data_ptr(), nbb.CaRule(), s)
dev.compact_load_dev(c, c2.data_ptr(), back.data_ptr(), 0, s)
res["ca_matches_int64_tile"] = bool(torch.equal(back, ref))
res["compact_bytes_per_pass"] = 3 ** r * 8
res["ca_compact_GBps"] = 2 * 3 ** r * 8 / (res["ca_compact_ms"] * 1e-3) / 1e9
print(json.dumps(res))
