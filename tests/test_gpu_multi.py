"""The reference's worker split over devices of one process (nbb_gpu_ca_multi /
nbb_gpu_reduction_multi): contiguous chunks of ceil(tiles / workers) compact tiles
(dispatch.cpp:416-432), halo cells read from the other workers' buffers inside the pass kernel
(peer memory), a flag barrier in device memory between passes. The result must be byte-identical
to the C oracle for any worker count (dispatch.hpp:103-107). With one GPU the workers share it
(separate buffers, the same peer-pointer reads and barrier); on a multi-GPU node the same calls
span devices."""
import numpy as np
import pytest

from _oracle import GASKET, orc_ca, orc_random_member_grid, orc_reduction
from paper_2004_13475_b200 import _abi, nbb
from paper_2004_13475_b200.nbb import CaRule, DispatchConfig, Grid

pytestmark = pytest.mark.gpu


def cfg(r, **kw):
    c = DispatchConfig(r=r, rho=32, max_cells=max(1 << 24, (1 << r) ** 2), device=0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def ndevices():
    return nbb.device_count()


@pytest.mark.parametrize("r,workers", [(5, 2), (8, 3), (10, 2), (10, 5), (12, 4), (13, 8)])
def test_ca_multi_matches_oracle(r, workers):
    devs = [w % ndevices() for w in range(workers)]
    init = orc_random_member_grid(r, 30 + r, 2)
    done, want = 0, init
    for steps in (1, 3, 8, 13):
        want = orc_ca(r, want, steps - done)
        done = steps
        got = nbb.run_ca_multi(cfg(r), devs, Grid(GASKET, r, init), steps)
        assert np.array_equal(got.grid.values, want), (r, workers, steps)
        assert len(got.reports) == steps


def test_ca_multi_rules_pass_lengths_and_pinned_io():
    """A generic rule, every pass length (pass_steps 1..12: the cluster walk's F = 8 and F = 12
    kernels over peer memory) and the zero-copy pinned host path."""
    torch = pytest.importorskip("torch")
    import ctypes
    r = 11
    devs = [0, 0, 0] if ndevices() == 1 else list(range(min(3, ndevices())))
    init = orc_random_member_grid(r, 5, 2)
    rule = CaRule(birth=(1 << 3) | (1 << 6), survive=(1 << 2) | (1 << 3))
    want = orc_ca(r, init, 9, rule.birth, rule.survive)
    for k in (1, 2, 3, 5, 8, 9, 12):
        got = nbb.run_ca_multi(cfg(r, pass_steps=k), devs, Grid(GASKET, r, init), 9, rule)
        assert np.array_equal(got.grid.values, want), k
    lib = _abi.load()
    h_in = torch.from_numpy(init.copy()).pin_memory()
    h_out = torch.zeros((1 << r, 1 << r), dtype=torch.int64).pin_memory()
    c = cfg(r, flags=_abi.FLAG_OUT_ZEROED).to_c()
    arr = (ctypes.c_int32 * len(devs))(*devs)
    assert lib.nbb_gpu_ca_multi(ctypes.byref(c), arr, len(devs), ctypes.c_void_p(h_in.data_ptr()), r, 9,
                                rule.birth, rule.survive, ctypes.c_void_p(h_out.data_ptr()), None) == 0
    assert np.array_equal(h_out.numpy(), want)


@pytest.mark.slow
def test_ca_multi_full_size_c3():
    """C3 (n = 2^16, seed 17) split over 2 workers, 20 steps: equal to the single-device run and
    to the reference's digest (tests/golden/c3_r16.json via the oracle pin)."""
    from _oracle import fnv1a64
    import json
    import os
    r = 16
    g = nbb.random_member_grid(GASKET, r, 17, 2, max_cells=1 << 32)
    one = nbb.run_ca(cfg(r), g, 20).grid.values
    d1 = fnv1a64(one)
    del one
    devs = [0, 0] if ndevices() == 1 else [0, 1]
    two = nbb.run_ca_multi(cfg(r), devs, g, 20).grid.values
    assert fnv1a64(two) == d1
    with open(os.path.join(os.path.dirname(__file__), "golden", "c3_r16.json")) as f:
        want = json.load(f)["trajectories"]["B3/S23"]["20"]
    assert int(two.sum()) == want["population"]


@pytest.mark.parametrize("r,workers", [(8, 2), (12, 3), (13, 5)])
def test_reduction_multi(r, workers):
    devs = [w % ndevices() for w in range(workers)]
    g = orc_random_member_grid(r, 1 + r, 100)
    assert nbb.run_reduction_multi(cfg(r), devs, Grid(GASKET, r, g)).value == orc_reduction(r, g)


def test_multi_rejects_bad_requests():
    r = 8
    g = Grid(GASKET, r, orc_random_member_grid(r, 1, 2))
    with pytest.raises(nbb.InvalidArgument):
        nbb.run_ca_multi(cfg(r), [0] * 9, g, 1)
    with pytest.raises(nbb.InvalidArgument):
        nbb.run_ca_multi(cfg(r), [0, 99], g, 1)
    with pytest.raises(nbb.InvalidArgument):
        nbb.run_ca_multi(cfg(r, mode=nbb.MapMode.BoundingBox), [0, 0], g, 1)
