"""Per-rank cost of the compact CA at N ranks, measured on ONE GPU (gpurun has 1 GPU).

For each level r in {16, 17} and N in {1, 2, 4, 8}, rank 0's shard (shard.compact_shard_chunk:
ceil(tiles / N) rounded up to whole cluster columns, dispatch.cpp:419-427) is advanced K steps by
the library's C++ pass loop:
  plain : the cluster pass kernel on the shard (nbb_gpu_ca_compact_passes_dev, no exchange)
          — the compute floor of one rank;
  p2p   : the P2P pass kernel on the shard (nbb_gpu_ca_compact_p2p_passes_dev) with world N and
          every peer mapped to this process (peer buffers and flags = ours, N arrivals per
          pass): the owner-by-ordinal halo path and the wait / arrive protocol all run; what a
          real N-GPU run adds is NVLink latency on the remote halo loads and the arrivals.
Both for one launch per step (`*_ms`, pass_steps 1) and for the default passes of up to 8
steps (`*_pass8_ms`). Prints one JSON line; ms per step = CUDA-event time / K.
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2004_13475_b200 import _abi, nbb, shard  # noqa: E402
from paper_2004_13475_b200 import device as dev  # noqa: E402

K = int(os.environ.get("K", "240"))
s = torch.cuda.current_stream().cuda_stream
lib = _abi.load()
out = {}


def timed(run):
    run(6)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(K)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / K


for r in (16, 17):
    members = 3 ** r
    c1 = torch.zeros(members, dtype=torch.int64, device="cuda")
    c1.random_(0, 2)
    c2 = torch.zeros_like(c1)
    base = nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2)
    for N in (1, 2, 4, 8):
        plan = shard.ShardPlan(r=r, rho=32, world=N, rank=0, state="compact")
        lc = plan.local_config(base)
        lc1 = plan.local_config(nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, pass_steps=1))
        t_plain = timed(lambda k: dev.ca_compact_passes_dev(lc1, c1.data_ptr(), c2.data_ptr(), k, nbb.CaRule(), s))
        t_plain2 = timed(lambda k: dev.ca_compact_passes_dev(lc, c1.data_ptr(), c2.data_ptr(), k, nbb.CaRule(), s))

        sync = torch.zeros(4, dtype=torch.int32, device="cuda")
        # every "peer" is this process: N entries pointing at our own buffers and sync word, so
        # the real owner table, phase split and barrier target (N arrivals per step) all run
        peer = [torch.tensor([b.data_ptr()] * N, dtype=torch.int64, device="cuda") for b in (c1, c2)]
        peer_flag = torch.tensor([sync.data_ptr()] * N, dtype=torch.int64, device="cuda")
        args = _abi.NbbP2P(N, 0, (ctypes.c_void_p * 2)(c1.data_ptr(), c2.data_ptr()),
                           (ctypes.c_void_p * 2)(peer[0].data_ptr(), peer[1].data_ptr()),
                           None, sync.data_ptr(), peer_flag.data_ptr(), 20000)
        cc = lc.to_c()
        st = {"i": 0}

        def p2p(k):
            rc = lib.nbb_gpu_ca_compact_p2p_dev(ctypes.byref(cc), st["i"], k, 8, 12, ctypes.byref(args),
                                                ctypes.c_void_p(s))
            assert rc == 0, lib.nbb_gpu_last_error()
            st["i"] += k

        def p2p2(k):  # passes of up to 8 steps
            rc = lib.nbb_gpu_ca_compact_p2p_passes_dev(ctypes.byref(cc), st["i"], k, 8, 12,
                                                       ctypes.byref(args), ctypes.c_void_p(s))
            assert rc == 0, lib.nbb_gpu_last_error()
            st["i"] += dev.pass_plan(lc, k).passes
        t_p2p = timed(p2p)
        t_p2p2 = timed(p2p2)
        torch.cuda.synchronize()
        assert int(sync[2].item()) == 0, "a wait timed out"
        assert int(sync[0].item()) == N * st["i"], (int(sync[0].item()), st["i"])
        out[f"r{r}_N{N}"] = {"tiles": plan.count, "plain_ms": t_plain, "p2p_world1_ms": t_p2p,
                             "plain_pass8_ms": t_plain2, "p2p_world1_pass8_ms": t_p2p2}
    one = out[f"r{r}_N1"]["plain_ms"]
    one2 = out[f"r{r}_N1"]["plain_pass8_ms"]
    for N in (1, 2, 4, 8):
        d = out[f"r{r}_N{N}"]
        d["ideal_ms"] = one / N
        d["efficiency_plain"] = one / N / d["plain_ms"]
        d["efficiency_p2p_world1"] = one / N / d["p2p_world1_ms"]
        d["efficiency_p2p_world1_pass8"] = one2 / N / d["p2p_world1_pass8_ms"]
    del c1, c2
print(json.dumps(out))
