"""Dataflow compact CA (all K steps in one launch, tile-level dependencies) vs one launch per
step: bit equality at several levels and step counts, then time at n = 2^16 / 2^17."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import device as dev  # noqa: E402
from paper_2004_13475_b200 import nbb  # noqa: E402

s = torch.cuda.current_stream().cuda_stream
res = {}


def cfgs(r):
    flow = nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2)
    tiles = 3 ** (r - 5)
    per_step = nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, shard_begin=0, shard_count=tiles)
    return flow, per_step


for r in (6, 10, 13, 16):
    flow, per_step = cfgs(r)
    g = torch.Generator(device="cuda")
    g.manual_seed(r)
    init = torch.randint(0, 2, (3 ** r,), dtype=torch.int64, device="cuda", generator=g)
    for K in (2, 3, 7, 20):
        a, b = init.clone(), torch.empty_like(init)
        dev.ca_compact_run_dev(flow, a.data_ptr(), b.data_ptr(), K, nbb.CaRule(), s)
        c, d = init.clone(), torch.empty_like(init)
        dev.ca_compact_run_dev(per_step, c.data_ptr(), d.data_ptr(), K, nbb.CaRule(), s)
        torch.cuda.synchronize()
        got, want = (b, d) if K % 2 else (a, c)
        res[f"r{r}_K{K}_equal"] = bool(torch.equal(got, want))


def timed(c, x, y, K):
    dev.ca_compact_run_dev(c, x.data_ptr(), y.data_ptr(), 10, nbb.CaRule(), s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dev.ca_compact_run_dev(c, x.data_ptr(), y.data_ptr(), K, nbb.CaRule(), s)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / K


for r in (16, 17):
    flow, per_step = cfgs(r)
    x = torch.randint(0, 2, (3 ** r,), dtype=torch.int64, device="cuda")
    y = torch.empty_like(x)
    res[f"r{r}_flow_ms"] = timed(flow, x, y, 200)
    res[f"r{r}_per_step_ms"] = timed(per_step, x, y, 200)
print(json.dumps(res))
