"""C4: the λ map over the level-16 orthotope, scalar K0 vs tensor-core K0-TC (for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import device as dev  # noqa: E402
from paper_2004_13475_b200 import nbb  # noqa: E402

lvl = int(os.environ.get("MAP_LEVEL", "16"))
s = torch.cuda.current_stream().cuda_stream
xy = torch.empty(3 ** lvl * 2, dtype=torch.int32, device="cuda")
for be in (nbb.LambdaBackend.Direct, nbb.LambdaBackend.MmaV2):
    c = nbb.DispatchConfig(r=16, rho=32, backend=be)
    for _ in range(2):
        dev.lambda_coords_dev(c, lvl, xy.data_ptr(), 4, s)
torch.cuda.synchronize()
