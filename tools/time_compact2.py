"""Two CA steps per pass (ca_compact2_kernel) vs one launch per step (ca_compact_kernel) on the
compact state: CUDA-event time of K steps through nbb_gpu_ca_compact_run_dev at n = 2^16, 2^17.

    python tools/time_compact2.py [K=200]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import _abi, nbb  # noqa: E402
from paper_2004_13475_b200 import device as dev  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
s = torch.cuda.current_stream().cuda_stream
for r in (16, 17):
    members = 3 ** r
    a = torch.randint(0, 2, (members,), dtype=torch.int64, device="cuda")
    b = torch.empty_like(a)
    highlife = nbb.CaRule(birth=(1 << 3) | (1 << 6), survive=(1 << 2) | (1 << 3))  # generic-rule kernel
    for name, flags, rule in (("pairs", 0, nbb.CaRule()), ("pairs_generic_rule", 0, highlife),
                              ("single", _abi.FLAG_SINGLE_STEP, nbb.CaRule())):
        c = nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, flags=flags)
        dev.ca_compact_run_dev(c, a.data_ptr(), b.data_ptr(), 20, rule, s)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dev.ca_compact_run_dev(c, a.data_ptr(), b.data_ptr(), K, rule, s)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / K)
        print(json.dumps({"r": r, "mode": name, "steps": K, "ms_per_step": best,
                          "Gcells_per_s": members / best / 1e6,
                          "GBps_state": (16 if name == "single" else 8) * members / best / 1e6}), flush=True)
    del a, b
