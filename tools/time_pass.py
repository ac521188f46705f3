"""K steps per pass over the compact state: CUDA-event time of S steps through
nbb_gpu_ca_compact_passes_dev (fewest passes) at n = 2^16 and 2^17, for the B3/S23
instantiation, a generic rule (B36/S23) and the bounding-box walk; results of every K checked
equal to K = 1 after 24 steps.

    python tools/time_pass.py [S=240] [K,K,...=1,2,3,4,6,8]
    NBB_PASS_IMPL=warp selects the warp-per-tile kernel (K <= 4); NBB_GPU_LIB a tuning build
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import nbb  # noqa: E402
from paper_2004_13475_b200 import device as dev  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 240
KS = [int(k) for k in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 3, 4, 6, 8]
s = torch.cuda.current_stream().cuda_stream
hl = nbb.CaRule(birth=(1 << 3) | (1 << 6), survive=(1 << 2) | (1 << 3))
for r in (16, 17):
    members = 3 ** r
    g = torch.Generator(device="cuda")
    g.manual_seed(r)
    a0 = torch.randint(0, 2, (members,), dtype=torch.int64, device="cuda", generator=g)
    a, b = torch.empty_like(a0), torch.empty_like(a0)
    ref = {}
    for K in KS:
        for name, rule, mode in (("conway", nbb.CaRule(), nbb.MapMode.Lambda), ("generic", hl, nbb.MapMode.Lambda),
                                 ("bb_conway", nbb.CaRule(), nbb.MapMode.BoundingBox)):
            c = nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, pass_steps=K, mode=mode)
            a.copy_(a0)
            st = dev.ca_compact_passes_dev(c, a.data_ptr(), b.data_ptr(), 24, rule, s)
            out = (b if st.result_in_b else a).clone()
            key = (name.replace("bb_", ""))
            same = None
            if K == 1 and key not in ref:
                ref[key] = out
            else:
                same = bool(torch.equal(out, ref[key]))
            dev.ca_compact_passes_dev(c, a.data_ptr(), b.data_ptr(), 4 * K, rule, s)
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                st = dev.ca_compact_passes_dev(c, a.data_ptr(), b.data_ptr(), S, rule, s)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            ms_pass = best / st.passes
            print(json.dumps({"r": r, "K": K, "mode": name, "steps": S, "passes": st.passes,
                              "ms_per_step": best / S, "ms_per_pass": ms_pass,
                              "GBps_per_pass": 16 * members / ms_pass / 1e6,
                              "Gcells_per_s": members * S / best / 1e6, "equal_to_K1": same}), flush=True)
    del a, b, a0
