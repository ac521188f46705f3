"""C4 at level 16: scalar K0, tcgen05 K0-TC and mma.sync K0-TC once each (for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import device as dev  # noqa: E402
from paper_2004_13475_b200 import nbb  # noqa: E402

s = torch.cuda.current_stream().cuda_stream
xy = torch.empty(3 ** 16 * 2, dtype=torch.int32, device="cuda")
for be in (nbb.LambdaBackend.Direct, nbb.LambdaBackend.MmaV2, nbb.LambdaBackend.MmaV1):
    dev.lambda_coords_dev(nbb.DispatchConfig(r=16, rho=32, backend=be), 16, xy.data_ptr(), 4, s)
torch.cuda.synchronize()
