"""Stress of the multi-GPU P2P step loop on one GPU: W ranks (processes time-sharing the GPU,
gloo for setup) run K compact CA steps through P2PCompactCA.run in chunks of random length
(exercising the arrival targets across calls), each rank's non-owned cells poisoned; the
gathered result must equal the single-GPU step loop. Prints one JSON line per configuration.

    python tools/p2p_stress.py
"""
import json
import os
import random
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, r, K, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2004_13475_b200 import nbb
    from paper_2004_13475_b200.shard import P2PCompactCA, ShardPlan
    plan = ShardPlan(r=r, rho=32, world=world, rank=rank, state="compact")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    init = torch.randint(0, 2, (3 ** r,), dtype=torch.int64, device="cuda", generator=gen)
    own = torch.zeros(3 ** r, dtype=torch.bool, device="cuda")
    for o, c in plan.compact_segments():
        own[o:o + c] = True
    init[~own] = 7
    ca = P2PCompactCA(plan, dist, device=0, timeout_ms=120000)
    ca.load(init)
    cfg = nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2)
    s = torch.cuda.current_stream().cuda_stream
    rng = random.Random(seed)  # the same chunking on every rank
    done = 0
    while done < K:
        k = min(K - done, rng.randint(1, 40))
        ca.run(cfg, nbb.CaRule(), k, s)
        done += k
    ca.check(s)
    out = torch.where(own, ca.state(), torch.zeros_like(ca.state())).cpu()
    ca.close()
    dist.all_reduce(out)
    if rank == 0:
        q.put(out.numpy())
    dist.destroy_process_group()


def main():
    from paper_2004_13475_b200 import device as dev
    from paper_2004_13475_b200 import nbb
    for world, r, K in ((2, 11, 301), (3, 12, 200), (4, 12, 150), (2, 14, 60), (3, 10, 500)):
        seed = 1000 * world + r
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _port()
        procs = [ctx.Process(target=worker, args=(i, world, port, r, K, seed, q)) for i in range(world)]
        for p in procs:
            p.start()
        got = q.get(timeout=1800)
        for p in procs:
            p.join(timeout=300)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(seed)
        a = torch.randint(0, 2, (3 ** r,), dtype=torch.int64, device="cuda", generator=gen)
        b = torch.empty_like(a)
        dev.ca_compact_run_dev(nbb.DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2), a.data_ptr(),
                               b.data_ptr(), K, nbb.CaRule(), torch.cuda.current_stream().cuda_stream)
        want = (b if K % 2 else a).cpu().numpy()
        print(json.dumps({"world": world, "r": r, "steps": K, "equal": bool(np.array_equal(got, want)),
                          "exitcodes": [p.exitcode for p in procs]}), flush=True)


if __name__ == "__main__":
    main()
