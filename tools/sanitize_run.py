"""Small end-to-end exercise of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck), checked against the C oracle:

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from _oracle import orc_ca, orc_random_member_grid, orc_reduction, orc_single_write  # noqa: E402
from paper_2004_13475_b200 import _abi, nbb  # noqa: E402

G = nbb.FractalSpec.sierpinski()
r = int(os.environ.get("SAN_R", "7"))
g = orc_random_member_grid(r, 5, 2)
want = orc_ca(r, g, 3)
checks = 0
for mode in (nbb.MapMode.Lambda, nbb.MapMode.BoundingBox):
    for rho in (8, 32):
        for kern in (nbb.KernelFamily.Tile, nbb.KernelFamily.PerCell):
            for cw in (8, 1, 0):
                if cw != 8 and (kern == nbb.KernelFamily.PerCell or rho != 32):
                    continue
                c = nbb.DispatchConfig(r=r, rho=rho, mode=mode, kernel=kern, cell_width=cw)
                assert np.array_equal(nbb.run_ca(c, nbb.Grid(G, r, g), 3).grid.values, want), (mode, rho, kern, cw)
                checks += 1
            c = nbb.DispatchConfig(r=r, rho=rho, mode=mode, kernel=kern)
            assert np.array_equal(nbb.run_single_write(c).grid.values, orc_single_write(r))
            assert nbb.run_reduction(c, nbb.Grid(G, r, g)).value == orc_reduction(r, g)
            checks += 2
for be in (nbb.LambdaBackend.MmaV1, nbb.LambdaBackend.MmaV2):
    c = nbb.DispatchConfig(r=r, rho=8, backend=be, kernel=nbb.KernelFamily.PerCell)
    assert np.array_equal(nbb.run_ca(c, nbb.Grid(G, r, g), 3).grid.values, want)
    checks += 1
for mode in (nbb.MapMode.Lambda, nbb.MapMode.BoundingBox):  # λ and BB launches over the compact state
    c = nbb.DispatchConfig(r=r, rho=32, mode=mode, flags=_abi.FLAG_COMPACT_STATE)
    assert np.array_equal(nbb.run_ca(c, nbb.Grid(G, r, g), 3).grid.values, want), mode
comp = nbb.compact_store(G, r, g)
assert np.array_equal(nbb.compact_load(G, comp, 0), g)
xy = nbb.lambda_coords(nbb.DispatchConfig(r=r, rho=1), r)
checks += 3
# zero-copy host buffers (pinned): member sectors read / written in place over PCIe
import ctypes  # noqa: E402
import torch  # noqa: E402
n = 1 << r
h_in = torch.from_numpy(g.copy()).pin_memory()
for fl, cw in ((_abi.FLAG_OUT_ZEROED, 8), (_abi.FLAG_OUT_ZEROED | _abi.FLAG_COMPACT_STATE, 8),
               (_abi.FLAG_OUT_ZEROED, 0)):
    h_out = torch.zeros((n, n), dtype=torch.int64).pin_memory()
    cc = nbb.DispatchConfig(r=r, rho=32, cell_width=cw, flags=fl).to_c()
    assert _abi.load().nbb_gpu_ca(ctypes.byref(cc), ctypes.c_void_p(h_in.data_ptr()), r, 3, 8, 12,
                                  ctypes.c_void_p(h_out.data_ptr()), None) == 0
    assert np.array_equal(h_out.numpy(), want), (fl, cw)
    checks += 1
# λ map kernels: scalar K0, tcgen05 K0-TC, mma.sync K0-TC
from _oracle import orc_lambda_coords  # noqa: E402
for be in (nbb.LambdaBackend.Direct, nbb.LambdaBackend.MmaV2, nbb.LambdaBackend.MmaV1):
    assert np.array_equal(nbb.lambda_coords(nbb.DispatchConfig(r=r, rho=1, backend=be), r),
                          orc_lambda_coords(r)), be
    checks += 1
# compact CA: the library's multi-step loop (PDL launches) and the P2P kernel (2-rank owner
# table and phase of rank 0, every peer mapped to this process)
from paper_2004_13475_b200 import device as dev, shard  # noqa: E402
cx, cy = orc_lambda_coords(r)[:, 0], orc_lambda_coords(r)[:, 1]
comp0 = torch.from_numpy(g[cy, cx].copy()).cuda()
ca, cb = comp0.clone(), torch.empty_like(comp0)
s = torch.cuda.current_stream().cuda_stream
cfg = nbb.DispatchConfig(r=r, rho=32)
dev.ca_compact_run_dev(cfg, ca.data_ptr(), cb.data_ptr(), 3, nbb.CaRule(), s)
assert np.array_equal(cb.cpu().numpy(), want[cy, cx])
checks += 1
# passes of 1..8 steps (ca_compact_sliced_kernel: TMA loader, named-barrier hand-off, halo
# gather), both rule instantiations, the λ and BB walks
for rule in (nbb.CaRule(), nbb.CaRule(birth=(1 << 3) | (1 << 6), survive=(1 << 2) | (1 << 3))):
    for k in (1, 2, 5, 8):
        for mode in (nbb.MapMode.Lambda, nbb.MapMode.BoundingBox):
            ca, cb = comp0.clone(), torch.empty_like(comp0)
            st = dev.ca_compact_passes_dev(nbb.DispatchConfig(r=r, rho=32, pass_steps=k, mode=mode), ca.data_ptr(),
                                           cb.data_ptr(), 11, rule, s)
            out = (cb if st.result_in_b else ca).cpu().numpy()
            assert np.array_equal(out, orc_ca(r, g, 11, rule.birth, rule.survive)[cy, cx]), (k, mode)
            checks += 1
# the P2P passes (world 2, rank 0; every peer mapped to this process): 8-step passes
plan = shard.ShardPlan(r=r, rho=32, world=2, rank=0, state="compact")
ca, cb = comp0.clone(), torch.zeros_like(comp0)  # rank 0 writes only its tiles
sync = torch.zeros(4, dtype=torch.int32, device="cuda")
peers = [torch.tensor([t.data_ptr()] * 2, dtype=torch.int64, device="cuda") for t in (ca, cb)]
flags = torch.tensor([sync.data_ptr()] * 2, dtype=torch.int64, device="cuda")
args = _abi.NbbP2P(2, 0, (ctypes.c_void_p * 2)(ca.data_ptr(), cb.data_ptr()),
                   (ctypes.c_void_p * 2)(peers[0].data_ptr(), peers[1].data_ptr()), None,
                   sync.data_ptr(), flags.data_ptr(), 20000)
cc = plan.local_config(cfg).to_c()
assert _abi.load().nbb_gpu_ca_compact_p2p_passes_dev(ctypes.byref(cc), 0, 8, 8, 12, ctypes.byref(args),
                                                     ctypes.c_void_p(s)) == 0
torch.cuda.synchronize()
own = plan.owner(plan.tile_of_ordinal(shard.lambda_inverse_blocks(cx >> 5, cy >> 5, plan.r_b, plan.W))) == 0
assert np.array_equal(cb.cpu().numpy()[own], orc_ca(r, g, 8)[cy, cx][own])
assert int(sync[0].item()) == 2 and int(sync[2].item()) == 0
checks += 1
# the worker split over devices (2 and 3 workers on this GPU)
for devs in ([0, 0], [0, 0, 0]):
    got = nbb.run_ca_multi(nbb.DispatchConfig(r=r, rho=32), devs, nbb.Grid(G, r, g), 9).grid.values
    assert np.array_equal(got, orc_ca(r, g, 9)), devs
    checks += 1
print(f"sanitize_run ok: r={r}, {checks} checks")
