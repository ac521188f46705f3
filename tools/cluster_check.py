"""Cluster walk (compact_cluster.cuh) vs the 32-ordinal sliced walk: bit-identical compact states
after S steps for every K = 1..12 (the sliced walk in passes of min(K, 8)) at r = 8..17 (random iid alive states, B3/S23 and B36/S23), and
the CUDA-event time of S steps with each walk at r = 16 / 17.

    python tools/cluster_check.py [S=24]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import nbb  # noqa: E402
from paper_2004_13475_b200 import device as dev  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 24
s = torch.cuda.current_stream().cuda_stream
hl = nbb.CaRule(birth=(1 << 3) | (1 << 6), survive=(1 << 2) | (1 << 3))


def run(impl, c, a0, steps, rule):
    os.environ["NBB_PASS_IMPL"] = impl
    a, b = a0.clone(), torch.empty_like(a0)
    st = dev.ca_compact_passes_dev(c, a.data_ptr(), b.data_ptr(), steps, rule, s)
    torch.cuda.synchronize()
    return b if st.result_in_b else a


bad = 0
for r in range(8, 18):
    g = torch.Generator(device="cuda")
    g.manual_seed(100 + r)
    a0 = torch.randint(0, 2, (3 ** r,), dtype=torch.int64, device="cuda", generator=g)
    for K in range(1, 13):
        for name, rule in (("conway", nbb.CaRule()), ("generic", hl)):
            c = nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, pass_steps=K)
            cs = nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, pass_steps=min(K, 8))
            x = run("sliced", cs, a0, S, rule)
            y = run("cluster", c, a0, S, rule)
            ok = bool(torch.equal(x, y))
            bad += not ok
            if not ok or K in (1, 8, 12):
                print(json.dumps({"r": r, "K": K, "rule": name, "steps": S, "equal": ok,
                                  "diff": int((x != y).sum())}), flush=True)
    del a0
for r in (16, 17):
    g = torch.Generator(device="cuda")
    g.manual_seed(r)
    a0 = torch.randint(0, 2, (3 ** r,), dtype=torch.int64, device="cuda", generator=g)
    a, b = a0.clone(), torch.empty_like(a0)
    for impl in ("sliced", "cluster"):
        os.environ["NBB_PASS_IMPL"] = impl
        for K in ((1, 4, 8) if impl == "sliced" else (1, 4, 8, 12)):
            for name, rule in (("conway", nbb.CaRule()), ("generic", hl)):
                c = nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, pass_steps=K)
                steps = 25 * K
                dev.ca_compact_passes_dev(c, a.data_ptr(), b.data_ptr(), 4 * K, rule, s)
                torch.cuda.synchronize()
                best = 1e9
                for _ in range(5):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    st = dev.ca_compact_passes_dev(c, a.data_ptr(), b.data_ptr(), steps, rule, s)
                    e1.record()
                    torch.cuda.synchronize()
                    best = min(best, e0.elapsed_time(e1))
                print(json.dumps({"r": r, "impl": impl, "K": K, "rule": name, "ms_per_step": best / steps,
                                  "ms_per_pass": best / st.passes,
                                  "GBps_per_pass": 16 * 3 ** r / (best / st.passes) / 1e6}), flush=True)
    del a, b, a0
print(json.dumps({"mismatching_cases": bad}))
