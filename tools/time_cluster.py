"""CUDA-event time of the compact CA pass at n = 2^16 (K = 1, 4, 8; B3/S23 and B36/S23) with the
library NBB_GPU_LIB (tuning builds), each result checked equal to the 32-ordinal sliced walk.

    NBB_GPU_LIB=tune/lib_x.so python tools/time_cluster.py [label]
(the sliced walk runs passes of min(K, 8); the comparison is after 3K steps)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import nbb  # noqa: E402
from paper_2004_13475_b200 import device as dev  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("NBB_GPU_LIB", "default")
s = torch.cuda.current_stream().cuda_stream
hl = nbb.CaRule(birth=(1 << 3) | (1 << 6), survive=(1 << 2) | (1 << 3))
r = int(os.environ.get("R", "16"))
g = torch.Generator(device="cuda")
g.manual_seed(r)
a0 = torch.randint(0, 2, (3 ** r,), dtype=torch.int64, device="cuda", generator=g)
a, b = a0.clone(), torch.empty_like(a0)
for K in (1, 4, 8, 10, 12):
    for name, rule in (("conway", nbb.CaRule()), ("generic", hl)):
        c = nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, pass_steps=K)
        outs = []
        for impl in ("sliced", "cluster"):
            os.environ["NBB_PASS_IMPL"] = impl
            a.copy_(a0)
            st = dev.ca_compact_passes_dev(c, a.data_ptr(), b.data_ptr(), 3 * K, rule, s)
            outs.append((b if st.result_in_b else a).clone())
        same = bool(torch.equal(outs[0], outs[1]))
        del outs
        steps = 25 * K
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = dev.ca_compact_passes_dev(c, a.data_ptr(), b.data_ptr(), steps, rule, s)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(json.dumps({"lib": label, "r": r, "K": K, "rule": name, "equal": same, "ms_per_step": round(best / steps, 5),
                          "ms_per_pass": round(best / st.passes, 4),
                          "frac_per_pass": round(16 * 3 ** r / (best / st.passes) / 1e6 / 6547.2, 3)}), flush=True)
