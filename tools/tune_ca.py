"""Time the CA step kernels for a given NBB_CA_PIPE setting (one process per setting,
since the choice is read once per process). Prints one JSON line per config.

    for p in 0 2,8 3,4 4,4 3,8; do NBB_CA_PIPE=$p python tools/tune_ca.py; done
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import device as dev  # noqa: E402
from paper_2004_13475_b200 import nbb  # noqa: E402


def main(r=16, K=50):
    n = 1 << r
    s = torch.cuda.current_stream().cuda_stream
    spec = nbb.FractalSpec.sierpinski()
    a = torch.zeros((n, n), dtype=torch.int64, device="cuda")
    vals = torch.from_numpy(nbb.random_member_values(spec, r, 17, 2)).cuda()
    base = nbb.DispatchConfig(r=r, rho=32, max_cells=n * n)
    dev.scatter_members_dev(base, vals.data_ptr(), a.data_ptr(), s)
    b = torch.zeros_like(a)
    a8 = torch.zeros((n, n), dtype=torch.uint8, device="cuda")
    b8 = torch.zeros_like(a8)
    dev.pack_alive_dev(nbb.DispatchConfig(r=r, rho=32, max_cells=n * n, cell_width=1), a.data_ptr(),
                       a8.data_ptr(), s)
    w1 = torch.zeros((n, n // 32), dtype=torch.int32, device="cuda")
    w2 = torch.zeros_like(w1)
    dev.pack_alive_dev(nbb.DispatchConfig(r=r, rho=32, max_cells=n * n, cell_width=0), a.data_ptr(),
                       w1.data_ptr(), s)
    out = {"pipe": os.environ.get("NBB_CA_PIPE", "default")}
    ref = None
    popcnt = lambda t: int(sum(bin(v & 0xFFFFFFFF).count("1") for v in t.view(-1).tolist()))  # noqa
    for name, kw, x, y in (("bit_lam32", dict(rho=32, cell_width=0), w1, w2),
                           ("bit_bb32", dict(rho=32, cell_width=0, mode=nbb.MapMode.BoundingBox), w1, w2),
                           ("i64_lam32", dict(rho=32), a, b), ("i64_lam16", dict(rho=16), a, b),
                           ("i64_lam8", dict(rho=8), a, b), ("u8_lam32", dict(rho=32, cell_width=1), a8, b8),
                           ("i64_bb32", dict(rho=32, mode=nbb.MapMode.BoundingBox), a, b),
                           ("u8_bb32", dict(rho=32, cell_width=1, mode=nbb.MapMode.BoundingBox), a8, b8)):
        c = nbb.DispatchConfig(r=r, max_cells=n * n, **kw)
        for _ in range(3):
            dev.ca_step_dev(c, x.data_ptr(), y.data_ptr(), nbb.CaRule(), s)
        torch.cuda.synchronize()
        if name.startswith("bit"):
            tmp = torch.zeros_like(a)
            dev.unpack_alive_dev(nbb.DispatchConfig(r=r, rho=32, max_cells=n * n, cell_width=0),
                                 y.data_ptr(), tmp.data_ptr(), s)
            chk = int(tmp.sum().item())
            del tmp
        else:
            chk = int(y.sum(dtype=torch.int64).item())
        ref = chk if ref is None else ref
        assert chk == ref, (name, chk, ref)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(K):
            dev.ca_step_dev(c, x.data_ptr(), y.data_ptr(), nbb.CaRule(), s)
        e1.record()
        e1.synchronize()
        out[name] = round(e0.elapsed_time(e1) / K, 4)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
