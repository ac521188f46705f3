import sys, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
from paper_2004_13475_b200 import nbb, device as dev
from _oracle import orc_lambda_coords
res = {}
for lvl in (1, 3, 8, 10, 13):
    want = orc_lambda_coords(lvl)
    for name, be in (("tc5", nbb.LambdaBackend.MmaV2),):
        got = nbb.lambda_coords(nbb.DispatchConfig(r=16, rho=32, backend=be), lvl)
        res[f"{name}_{lvl}"] = bool(np.array_equal(got, want))
        if not res[f"{name}_{lvl}"]:
            bad = np.nonzero((got != want).any(1))[0]
            res[f"{name}_{lvl}_bad"] = [int(bad.size), got[bad[:3]].tolist(), want[bad[:3]].tolist()]
print(json.dumps(res))
s = torch.cuda.current_stream().cuda_stream
xy = torch.empty(3 ** 16 * 2, dtype=torch.int32, device="cuda")
for name, be in (("scalar", nbb.LambdaBackend.Direct), ("tc5", nbb.LambdaBackend.MmaV2), ("mmasync", nbb.LambdaBackend.MmaV1)):
    c = nbb.DispatchConfig(r=16, rho=32, backend=be)
    for _ in range(3): dev.lambda_coords_dev(c, 16, xy.data_ptr(), 4, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): dev.lambda_coords_dev(c, 16, xy.data_ptr(), 4, s)
    e1.record(); e1.synchronize()
    print(name, e0.elapsed_time(e1) / 20, "ms at level 16")
