"""The multi-process compact CA over the library's NCCL communicator (nbb_gpu_comm_*): on one GPU
a single-rank communicator (the pass loop, reduction and NCCL binding through the same entry
points); with >= 2 GPUs, 2 ranks under torchrun exchange real halos. Bit-exact with the C oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

from _oracle import ROOT, orc_ca_compact, orc_random_member_compact
from paper_2004_13475_b200 import nbb, shard
from paper_2004_13475_b200.nbb import CaRule, DispatchConfig

pytestmark = pytest.mark.gpu


def cfg(r, **kw):
    c = DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, device=0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def test_single_rank_comm_matches_oracle():
    import torch
    r = 13
    s = torch.cuda.current_stream().cuda_stream
    c0 = orc_random_member_compact(r, 14, 2)
    ca = shard.NcclCompactCA(r, None, 0)
    try:
        ca.load(torch.from_numpy(c0))
        want, done = c0, 0
        for steps in (3, 8, 20):
            ca.run(cfg(r), CaRule(), steps - done, s)
            want = orc_ca_compact(r, want, steps - done)
            done = steps
            assert np.array_equal(ca.state().cpu().numpy(), want), steps
        assert ca.reduction(cfg(r), s) == int(want.sum())
    finally:
        ca.close()


WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["NBB_ROOT"]); sys.path.insert(0, os.path.join(os.environ["NBB_ROOT"], "tests"))
import numpy as np, torch, torch.distributed as dist
from _oracle import orc_ca_compact, orc_random_member_compact
from paper_2004_13475_b200 import shard
from paper_2004_13475_b200.nbb import CaRule, DispatchConfig
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
r = int(os.environ["NBB_R"]); s = torch.cuda.current_stream().cuda_stream
c0 = orc_random_member_compact(r, 21, 2)
ca = shard.NcclCompactCA(r, dist, rank)
ca.load(torch.from_numpy(c0))
cfg = DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, device=rank)
ca.run(cfg, CaRule(), 11, s)
plan = shard.ShardPlan(r=r, rho=32, world=world, rank=rank, state="compact")
want = orc_ca_compact(r, c0, 11)
got = ca.state().cpu().numpy()
for off, cnt in plan.compact_segments():
    assert np.array_equal(got[off:off + cnt], want[off:off + cnt]), (rank, off)
assert ca.reduction(cfg, s) == int(want.sum())
ca.close(); dist.destroy_process_group()
print("rank", rank, "ok")
'''


@pytest.mark.skipif("not __import__('torch').cuda.device_count() >= 2", reason="needs 2 GPUs")
@pytest.mark.parametrize("r", [10, 13])
def test_two_rank_comm_matches_oracle(tmp_path, r):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, NBB_ROOT=ROOT, NBB_R=str(r))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr", "127.0.0.1", "--master-port", "29561", str(script)],
                         env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert out.stdout.count("ok") == 2
