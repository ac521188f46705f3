"""GPU parity: every kernel family against the C oracle / the reference's golden
outputs, bit-exact (integer and byte work). Run on a B200 with `pytest -m gpu`."""
import itertools
import os
import subprocess

import numpy as np
import pytest

from _oracle import (GASKET, ROOT, fnv1a64, orc_ca, orc_ca_compact_check, orc_lambda_coords,
                     orc_random_member_grid, orc_reduction, orc_single_write)
from paper_2004_13475_b200 import _abi, nbb
from paper_2004_13475_b200.nbb import (CaRule, DispatchConfig, Grid, IntraBlockStrategy,
                                       KernelFamily, LambdaBackend, MapMode)

pytestmark = pytest.mark.gpu

B3S23 = CaRule()


def cfg(**kw):
    c = DispatchConfig()
    for k, v in kw.items():
        setattr(c, k, v)
    n = c.spec.side_length(c.r)
    c.max_cells = max(c.max_cells, n * n)
    return c


def grid(values, r):
    return Grid(GASKET, r, np.ascontiguousarray(values, dtype=np.int64))


def nonmember_mask(r):
    n = 1 << r
    yy, xx = np.mgrid[0:n, 0:n]
    return (xx & (n - 1 - yy)) != 0


def with_garbage(values, r, seed=0):
    g = values.copy()
    m = nonmember_mask(r)
    rng = np.random.default_rng(seed)
    g[m] = rng.integers(-2**62, 2**62, size=int(m.sum()))
    return g


KERNEL_COMBOS = [  # (mode, rho, kernel, cell_width)
    (MapMode.Lambda, rho, k, cw)
    for rho in (1, 2, 4, 8, 16, 32) for k in (KernelFamily.Auto, KernelFamily.PerCell)
    for cw in (8, 1)
] + [(MapMode.BoundingBox, rho, k, cw)
     for rho in (1, 2, 4, 8, 16, 32) for k in (KernelFamily.Auto, KernelFamily.PerCell)
     for cw in (8, 1)
] + [(mode, rho, KernelFamily.Tile, 8)  # the embedded int64 tile kernels (Auto takes the compact state)
     for mode in (MapMode.Lambda, MapMode.BoundingBox) for rho in (8, 16, 32)]


def test_device_present():
    assert nbb.device_count() >= 1


@pytest.mark.parametrize("r", [0, 1, 2, 3, 5, 6, 8, 10])
def test_single_write(r):
    want = orc_single_write(r)
    for mode, rho, k, _ in KERNEL_COMBOS:
        if (1 << r) % rho:
            continue
        got = nbb.run_single_write(cfg(r=r, rho=rho, mode=mode, kernel=k))
        assert np.array_equal(got.grid.values, want), (mode, rho, k)
        assert got.report.csv_row() == nbb.plan_report(cfg(r=r, rho=rho, mode=mode)).csv_row()


@pytest.mark.parametrize("r", [0, 2, 4, 5, 7, 9, 10])
def test_reduction_ignores_nonmember_garbage(r):
    g = with_garbage(orc_random_member_grid(r, 5 + r, 1 << 40), r, seed=r)
    want = orc_reduction(r, g)
    for mode, rho, k, cw in KERNEL_COMBOS:
        if (1 << r) % rho or cw != 8:
            continue
        got = nbb.run_reduction(cfg(r=r, rho=rho, mode=mode, kernel=k), grid(g, r))
        assert got.value == want, (mode, rho, k)


def test_reduction_wraps_like_int64():
    r = 6
    g = orc_random_member_grid(r, 3, 2)
    g[g == 1] = 2**62 + 12345  # sum overflows int64: must wrap identically
    assert nbb.run_reduction(cfg(r=r, rho=8), grid(g, r)).value == orc_reduction(r, g)


RULES = [CaRule(), CaRule(birth=(1 << 3) | (1 << 6), survive=(1 << 2) | (1 << 3)),
         CaRule(birth=1 << 2, survive=0), CaRule(birth=0x1FF, survive=0x1FF),
         CaRule(birth=1 | (1 << 8), survive=(1 << 1) | (1 << 8)), CaRule(birth=0, survive=0)]


@pytest.mark.parametrize("r", [1, 2, 3, 5, 6, 8, 9])
def test_ca_all_kernels(r):
    init = with_garbage(orc_random_member_grid(r, 40 + r, 2), r, seed=r) if r >= 2 else \
        orc_random_member_grid(r, 40 + r, 2)
    for rule in RULES[:3] if r > 6 else RULES:
        for steps in (1, 3):
            want = orc_ca(r, init, steps, rule.birth, rule.survive)
            for mode, rho, k, cw in KERNEL_COMBOS:
                if (1 << r) % rho:
                    continue
                got = nbb.run_ca(cfg(r=r, rho=rho, mode=mode, kernel=k, cell_width=cw),
                                 grid(init, r), steps, rule)
                assert np.array_equal(got.grid.values, want), (mode, rho, k, cw, rule, steps)
                assert len(got.reports) == steps
                assert got.grid.generation() == steps


@pytest.mark.parametrize("r", [5, 6, 8, 10, 12])
def test_ca_bit_packed_state(golden, r):
    """cell_width 0: the alive state is one bit per cell (exact: CA reads != 0, writes 0/1)."""
    init = with_garbage(orc_random_member_grid(r, 90 + r, 2), r, seed=r) if r <= 10 else \
        orc_random_member_grid(r, 90 + r, 2)
    for rule in (RULES[:4] if r <= 8 else RULES[:1]):
        for steps in (1, 2, 7):
            want = orc_ca(r, init, steps, rule.birth, rule.survive)
            for mode in (MapMode.Lambda, MapMode.BoundingBox):
                got = nbb.run_ca(cfg(r=r, rho=32, mode=mode, cell_width=0), grid(init, r), steps, rule)
                assert np.array_equal(got.grid.values, want), (r, mode, rule, steps)
    if r >= 10:
        w = golden["workloads"][str(r)]
        g = nbb.random_member_grid(GASKET, r, 1 + r, 2, max_cells=1 << (2 * r))
        for k, (pop, digest) in w["ca"].items():
            out = nbb.run_ca(cfg(r=r, rho=32, cell_width=0), g, int(k)).grid.values
            assert (int(out.sum()), fnv1a64(out)) == (pop, digest), k
    with pytest.raises(nbb.InvalidArgument, match="1-bit packed"):
        nbb.run_ca(cfg(r=r, rho=16, cell_width=0), grid(init, r), 1)


@pytest.mark.parametrize("cw,state", [(8, 0), (8, _abi.FLAG_EMBEDDED_STATE), (1, 0), (0, 0),
                                      (8, _abi.FLAG_COMPACT_STATE)])
def test_ca_host_buffers_pinned_zero_copy(cw, state):
    """nbb_gpu_ca on pinned host buffers: member sectors move in place over PCIe; with
    FLAG_OUT_ZEROED only member cells of out are written; without it out is written whole."""
    torch = pytest.importorskip("torch")
    import ctypes
    r, n = 11, 1 << 11
    init = with_garbage(orc_random_member_grid(r, 77, 2), r, seed=5)
    want = orc_ca(r, init, 5)
    lib = _abi.load()
    h_in = torch.from_numpy(init.copy()).pin_memory()
    for flags, out_init in ((_abi.FLAG_OUT_ZEROED, 0), (0, 0), (0, 7)):
        h_out = torch.full((n, n), out_init, dtype=torch.int64).pin_memory()
        c = cfg(r=r, rho=32, cell_width=cw, flags=flags | state).to_c()
        rc = lib.nbb_gpu_ca(ctypes.byref(c), ctypes.c_void_p(h_in.data_ptr()), r, 5, 8, 12,
                            ctypes.c_void_p(h_out.data_ptr()), None)
        assert rc == 0, lib.nbb_gpu_last_error()
        assert np.array_equal(h_out.numpy(), want), (cw, flags, out_init)
    assert np.array_equal(h_in.numpy(), init)  # the input is never written
    # in place (out aliases the pinned input): full write, garbage cleared
    h_io = torch.from_numpy(init.copy()).pin_memory()
    c = cfg(r=r, rho=32, cell_width=cw, flags=state).to_c()
    assert lib.nbb_gpu_ca(ctypes.byref(c), ctypes.c_void_p(h_io.data_ptr()), r, 5, 8, 12,
                          ctypes.c_void_p(h_io.data_ptr()), None) == 0
    assert np.array_equal(h_io.numpy(), want)


def test_ca_semantics_probes():
    """App. B.4: steps=0 returns the input unchanged (garbage included); alive means != 0."""
    r = 6
    g = with_garbage(orc_random_member_grid(r, 1, 2), r)
    c = cfg(r=r, rho=8)
    assert np.array_equal(nbb.run_ca(c, grid(g, r), 0).grid.values, g)
    g5 = orc_random_member_grid(r, 1, 2)
    a = nbb.run_ca(c, grid(g5 * 5, r), 4).grid.values
    assert np.array_equal(a, nbb.run_ca(c, grid(g5, r), 4).grid.values)
    dead = np.zeros_like(g5)
    assert not nbb.run_ca(c, grid(dead, r), 3).grid.values.any()
    lonely = dead.copy()
    lonely[0, 0] = 1
    assert not nbb.run_ca(c, grid(lonely, r), 1).grid.values.any()


def test_reference_pins(golden):
    p = golden["pins"]
    for seed in (1234, 2024):
        g = orc_random_member_grid(5, seed, 2)
        for rho, mode in ((1, MapMode.Lambda), (8, MapMode.Lambda), (32, MapMode.Lambda),
                          (1, MapMode.BoundingBox), (32, MapMode.BoundingBox)):
            for steps in (1, 4, 10):
                out = nbb.run_ca(cfg(r=5, rho=rho, mode=mode), grid(g, 5), steps).grid.values
                assert fnv1a64(out) == p[f"ca_r5_seed{seed}"]["steps"][steps], (seed, rho, steps)
    g = orc_random_member_grid(5, 99, 1000)
    assert nbb.run_reduction(cfg(r=5, rho=4), grid(g, 5)).value == p["rd_r5_seed99_mod1000"]


def test_mode_equivalence_matrix(golden):
    """acceptance.cpp:153-208 — every valid (rho, strategy, backend) computes the same
    SW grid, RD value and 2-step CA grid as the reference, r <= 8."""
    for r in range(0, 9):
        w = golden["workloads"][str(r)]
        rd = orc_random_member_grid(r, 17 + r, 100)
        ca = orc_random_member_grid(r, 71 + r, 2)
        combos = 0
        for rho, st, be in itertools.product((1, 2, 4, 8, 16), IntraBlockStrategy, LambdaBackend):
            c = cfg(r=r, rho=rho, strategy=st, backend=be)
            try:
                c.validate()
            except nbb.InvalidArgument:
                continue
            tag = (r, rho, st.name, be.name)
            assert fnv1a64(nbb.run_single_write(c).grid.values) == w["sw_fnv"], tag
            assert nbb.run_reduction(c, grid(rd, r)).value == w["acceptance_rd_value"], tag
            assert fnv1a64(nbb.run_ca(c, grid(ca, r), 2).grid.values) == w["acceptance_ca2_fnv"], tag
            c.flags = _abi.FLAG_EMBEDDED_STATE  # the embedded grid with this (strategy, backend)
            assert fnv1a64(nbb.run_ca(c, grid(ca, r), 2).grid.values) == w["acceptance_ca2_fnv"], tag
            combos += 1
        assert combos > 0


@pytest.mark.parametrize("r", [11, 12, 13, 14])
def test_golden_workloads_tile_path(golden, r):
    w = golden["workloads"][str(r)]
    for rho in (8, 16, 32):
        for mode in (MapMode.Lambda, MapMode.BoundingBox):
            c = cfg(r=r, rho=rho, mode=mode, kernel=KernelFamily.Tile)
            assert fnv1a64(nbb.run_single_write(c).grid.values) == w["sw_fnv"], (rho, mode)
    g = nbb.random_member_grid(GASKET, r, 1 + r, 100, max_cells=1 << (2 * r))
    assert fnv1a64(g.values) == w["rd_grid_fnv"]
    for rho in (8, 16, 32):
        assert nbb.run_reduction(cfg(r=r, rho=rho, kernel=KernelFamily.Tile), g).value == w["rd_value"]
    g = nbb.random_member_grid(GASKET, r, 1 + r, 2, max_cells=1 << (2 * r))
    for rho, cw, mode in ((32, 8, MapMode.Lambda), (16, 8, MapMode.Lambda), (8, 8, MapMode.Lambda),
                          (32, 1, MapMode.Lambda), (32, 8, MapMode.BoundingBox),
                          (32, 1, MapMode.BoundingBox)):
        c = cfg(r=r, rho=rho, mode=mode, cell_width=cw, kernel=KernelFamily.Tile)
        for k, (pop, digest) in w["ca"].items():
            out = nbb.run_ca(c, g, int(k)).grid.values
            assert (int(out.sum()), fnv1a64(out)) == (pop, digest), (rho, cw, mode, k)


def test_lambda_coords_map_kernels(golden):
    for level in range(0, 16):
        want = golden["lambda_digests"][str(level)]
        assert fnv1a64(nbb.lambda_coords(cfg(r=level), level)) == want, level
        if level <= 16:  # K0-TC: mma.sync (MmaV1) and tcgen05 + TMEM (MmaV2)
            for be in (LambdaBackend.MmaV1, LambdaBackend.MmaV2):
                got = nbb.lambda_coords(cfg(r=level, backend=be), level)
                assert fnv1a64(got) == want, ("tc", be, level)
    assert np.array_equal(nbb.lambda_coords(cfg(), 9), orc_lambda_coords(9))


@pytest.mark.parametrize("level", [11, 13, 16, 17])
def test_lambda_map_full_levels(level):
    """K0 over whole orthotopes up to the C4 sweep's top level (row carries at W = 3^⌈L/2⌉,
    the 729-entry digit carries, a quad tail when 3^L is odd): int32 pairs on the device and
    int64 pairs through the host call, bit-exact against the C oracle."""
    import torch
    from paper_2004_13475_b200 import device as dev
    want = orc_lambda_coords(level)
    s = torch.cuda.current_stream().cuda_stream
    xy = torch.empty((3 ** level, 2), dtype=torch.int32, device="cuda")
    dev.lambda_coords_dev(cfg(), level, xy.data_ptr(), 4, s)
    assert np.array_equal(xy.cpu().numpy().astype(np.int64), want)
    # the tcgen05 K0-TC at full size too (int32 pairs, levels <= 17)
    dev.lambda_coords_dev(cfg(backend=LambdaBackend.MmaV2), level, xy.data_ptr(), 4, s)
    assert np.array_equal(xy.cpu().numpy().astype(np.int64), want)
    del xy
    assert np.array_equal(nbb.lambda_coords(cfg(), level), want)


def test_workers_shard_the_ordinal_range():
    """Contiguous ordinal chunks (dispatch.cpp:419-427) give identical results for any count."""
    r = 9
    g = orc_random_member_grid(r, 8, 2)
    v = orc_random_member_grid(r, 8, 50)
    base = None
    for workers in (1, 2, 3, 5, 8):
        c = cfg(r=r, rho=16, workers=workers)
        out = (fnv1a64(nbb.run_single_write(c).grid.values), nbb.run_reduction(c, grid(v, r)).value,
               fnv1a64(nbb.run_ca(c, grid(g, r), 4).grid.values))
        base = base or out
        assert out == base, workers


def test_timing_reports_micros():
    r = 10
    c = cfg(r=r, rho=32, timing=True)
    res = nbb.run_ca(c, grid(orc_random_member_grid(r, 1, 2), r), 2)
    assert all(rep.micros >= 0 for rep in res.reports)
    assert nbb.run_single_write(cfg(r=r, rho=32)).report.micros == 0


def test_device_resident_api():
    torch = pytest.importorskip("torch")
    from paper_2004_13475_b200 import device as dev
    r = 12
    n = 1 << r
    c = cfg(r=r, rho=32)
    values = nbb.random_member_values(GASKET, r, 13, 2)
    d_vals = torch.from_numpy(values).cuda()
    a = torch.zeros((n, n), dtype=torch.int64, device="cuda")
    b = torch.zeros_like(a)
    s = torch.cuda.current_stream().cuda_stream
    dev.scatter_members_dev(c, d_vals.data_ptr(), a.data_ptr(), s)
    host = nbb.random_member_grid(GASKET, r, 13, 2)
    assert np.array_equal(a.cpu().numpy(), host.values)
    want = orc_ca(r, host.values, 3)
    for _ in range(3):
        dev.ca_step_dev(c, a.data_ptr(), b.data_ptr(), CaRule(), s)
        a, b = b, a
    assert np.array_equal(a.cpu().numpy(), want)
    # uint8 state path: pack -> steps -> unpack
    a8 = torch.zeros((n, n), dtype=torch.uint8, device="cuda")
    b8 = torch.zeros_like(a8)
    g64 = torch.from_numpy(with_garbage(host.values, r)).cuda()
    c8 = cfg(r=r, rho=32, cell_width=1)
    dev.pack_alive_dev(c8, g64.data_ptr(), a8.data_ptr(), s)
    for _ in range(3):
        dev.ca_step_dev(c8, a8.data_ptr(), b8.data_ptr(), CaRule(), s)
        a8, b8 = b8, a8
    out64 = torch.empty_like(g64)
    dev.unpack_alive_dev(c8, a8.data_ptr(), out64.data_ptr(), s)
    assert np.array_equal(out64.cpu().numpy(), want)
    # sanitize zeroes exactly the non-members
    gg = torch.from_numpy(with_garbage(host.values, r)).cuda()
    dev.sanitize_dev(c, gg.data_ptr(), s)
    assert np.array_equal(gg.cpu().numpy(), host.values)
    # reduction into device memory
    val = torch.zeros(1, dtype=torch.int64, device="cuda")
    hv = nbb.random_member_grid(GASKET, r, 5, 1000)
    dv = torch.from_numpy(hv.values).cuda()
    dev.reduction_dev(c, dv.data_ptr(), val.data_ptr(), s)
    assert int(val.item()) == orc_reduction(r, hv.values)
    # map kernel into device memory, int32 pairs
    xy = torch.empty((3 ** 10, 2), dtype=torch.int32, device="cuda")
    dev.lambda_coords_dev(c, 10, xy.data_ptr(), 4, s)
    assert np.array_equal(xy.cpu().numpy().astype(np.int64), orc_lambda_coords(10))


@pytest.mark.parametrize("name", ["vicsek", "carpet"])
def test_generic_specs(golden, name):
    """Vicsek (k=5, s=3) and carpet (k=8, s=3) through the table-driven per-cell kernels:
    every valid (mode, strategy, backend) reproduces the reference's SW / RD / 2-step CA
    (acceptance.cpp:153-208 for all specs) and λ (criterion 1)."""
    from paper_2004_13475_b200.nbb import FractalSpec
    spec = FractalSpec.builtin(name)
    for r in range(0, 6):
        w = golden["generic_specs"][name][str(r)]
        n = spec.side_length(r)
        rd = nbb.random_member_grid(spec, r, 17 + r, 100)
        ca = nbb.random_member_grid(spec, r, 71 + r, 2)
        assert fnv1a64(rd.values) == w["rd_grid_fnv"] and fnv1a64(ca.values) == w["ca_grid_fnv"]
        combos = 0
        for mode, st, be in itertools.product(MapMode, IntraBlockStrategy, LambdaBackend):
            c = DispatchConfig(spec=spec, r=r, rho=1, mode=mode, strategy=st, backend=be,
                               max_cells=max(1 << 24, n * n))
            try:
                c.validate()
            except nbb.InvalidArgument:
                continue
            tag = (name, r, mode.name, st.name, be.name)
            assert fnv1a64(nbb.run_single_write(c).grid.values) == w["sw_fnv"], tag
            assert nbb.run_reduction(c, rd).value == w["rd_value"], tag
            assert fnv1a64(nbb.run_ca(c, ca, 2).grid.values) == w["ca2_fnv"], tag
            combos += 1
        assert combos >= 4
        assert fnv1a64(nbb.lambda_coords(DispatchConfig(spec=spec), r)) == w["lambda_fnv"], r


def test_compact_codec_matches_reference():
    """compact_store / compact_load (block_map.cpp:245-282) and λ⁻¹ (:113-148) on the device,
    against the reference library (criterion 7: round trip, k^r slots)."""
    import ctypes
    from _oracle import ref_available, ref_lib
    from paper_2004_13475_b200.nbb import FractalSpec
    for spec, rmax in ((GASKET, 10), (FractalSpec.vicsek(), 5), (FractalSpec.carpet(), 4)):
        for r in range(0, rmax + 1):
            n = spec.side_length(r)
            dense = nbb.random_member_grid(spec, r, 1234 + r, 100000, max_cells=max(1 << 24, n * n)).values
            comp = nbb.compact_store(spec, r, dense)
            assert comp.size() == spec.volume(r)
            if ref_available():
                want = np.empty(spec.volume(r), dtype=np.int64)
                assert ref_lib().ref_compact_store(ctypes.byref(spec.to_c()), r,
                                                   dense.ctypes.data_as(ctypes.c_void_p),
                                                   want.ctypes.data_as(ctypes.c_void_p)) == 0
                assert np.array_equal(comp.values.ravel(), want), (spec.name, r)
            assert np.array_equal(nbb.compact_load(spec, comp, 0), dense), (spec.name, r)
            full = nbb.compact_load(spec, comp, -7)
            assert np.count_nonzero(full == -7) >= n * n - spec.volume(r)
    # λ⁻¹ round trip and the reference's errors
    xy = nbb.lambda_coords(cfg(), 9)
    om = nbb.lambda_inverse(GASKET, 9, xy)
    w = 3 ** 5
    assert np.array_equal(om[:, 1] * w + om[:, 0], np.arange(3 ** 9))
    with pytest.raises(nbb.DomainError, match="is not a member cell at level 2"):
        nbb.lambda_inverse(GASKET, 2, [(0, 0), (1, 0)])
    with pytest.raises(nbb.OutOfRange, match="outside 4\\^2"):
        nbb.lambda_inverse(GASKET, 2, [(4, 0)])


@pytest.mark.parametrize("r", [5, 6, 9, 12])
def test_ca_compact_state(golden, r):
    """NBB_FLAG_COMPACT_STATE: the CA state lives in the λ-ordered compact layout on the
    device (ca_compact_kernel); results equal the oracle / the reference's golden."""
    from paper_2004_13475_b200 import _abi as abi
    init = with_garbage(orc_random_member_grid(r, 50 + r, 2), r, seed=r) if r <= 9 else \
        orc_random_member_grid(r, 50 + r, 2)
    for rule in (RULES[:4] if r <= 6 else RULES[:1]):
        for steps in (1, 3, 10):
            want = orc_ca(r, init, steps, rule.birth, rule.survive)
            got = nbb.run_ca(cfg(r=r, rho=32, flags=abi.FLAG_COMPACT_STATE), grid(init, r), steps, rule)
            assert np.array_equal(got.grid.values, want), (r, rule, steps)
    w = golden["workloads"][str(r)]
    g = nbb.random_member_grid(GASKET, r, 1 + r, 2, max_cells=1 << (2 * r))
    for k, (pop, digest) in w["ca"].items():
        out = nbb.run_ca(cfg(r=r, rho=32, flags=abi.FLAG_COMPACT_STATE), g, int(k)).grid.values
        assert (int(out.sum()), fnv1a64(out)) == (pop, digest), k
    # the bounding-box launch over the same compact state (box tiles culled, λ⁻¹ addressing)
    for steps in (1, 4):
        out = nbb.run_ca(cfg(r=r, rho=32, mode=MapMode.BoundingBox, flags=abi.FLAG_COMPACT_STATE), g,
                         steps).grid.values
        assert (int(out.sum()), fnv1a64(out)) == tuple(w["ca"][str(steps)]), ("bb", steps)


def test_compact_device_workloads():
    torch = pytest.importorskip("torch")
    from paper_2004_13475_b200 import device as dev
    r = 12
    c = cfg(r=r, rho=32)
    s = torch.cuda.current_stream().cuda_stream
    host = nbb.random_member_grid(GASKET, r, 5, 1000)
    emb = torch.from_numpy(host.values).cuda()
    comp = torch.empty(3 ** r, dtype=torch.int64, device="cuda")
    dev.compact_store_dev(c, emb.data_ptr(), comp.data_ptr(), s)
    val = torch.zeros(1, dtype=torch.int64, device="cuda")
    dev.reduction_compact_dev(c, comp.data_ptr(), val.data_ptr(), s)
    assert int(val.item()) == orc_reduction(r, host.values)
    dev.single_write_compact_dev(c, comp.data_ptr(), s)
    back = torch.zeros_like(emb)
    dev.compact_load_dev(c, comp.data_ptr(), back.data_ptr(), 0, s)
    assert np.array_equal(back.cpu().numpy(), orc_single_write(r))


def test_nbbmap_bench_csv_byte_identical(golden, tmp_path):
    """`nbbmap bench` over the GPU path prints the reference CLI's CSV bytes
    (tools/nbbmap.cpp:530-625; test_cli.cpp:151-175), for any worker count."""
    from paper_2004_13475_b200 import nbbmap
    for case in golden["cli_bench"]:
        for extra in ([], ["--workers", "4"]):
            out = tmp_path / "b.csv"
            rc = nbbmap.main(case["args"].split() + extra + ["--out", str(out)])
            assert rc == 0, case["args"]
            assert out.read_text() == case["csv"], (case["args"], extra)
    out = tmp_path / "t.csv"
    assert nbbmap.main("bench --workload ca --rmin 10 --rmax 10 --rho 32 --timing --out".split() +
                       [str(out)]) == 0
    rows = out.read_text().splitlines()[1:]
    assert len(rows) == 2 and all(int(r.split(",")[11]) >= 0 for r in rows)
    assert nbbmap.main("bench --rmin 13 --rmax 13".split()) == 3  # --max-cells budget


def test_cpp_shim_on_gpu():
    src = os.path.join(ROOT, "tests", "cpp", "shim_example.cpp")
    out = "/tmp/nbb_shim_example_gpu"
    libdir = os.path.dirname(_abi.LIB_PATH)
    subprocess.run(["/usr/bin/g++", "-std=c++17", f"-I{os.path.join(ROOT, 'include')}", src, "-o", out,
                    f"-L{libdir}", "-lnbbgpu", f"-Wl,-rpath,{libdir}"], check=True)
    r = subprocess.run([out], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ca pop 10398" in r.stdout
    # nbb::gpu::run_ca (the reference signature) at n = 2^13, 20 steps: default (compact) state,
    # compact with 3 steps per pass, embedded int64 grid — all equal the C oracle
    want = fnv1a64(orc_ca(13, orc_random_member_grid(13, 14, 2), 20))
    for tag in ("default", "compact3", "embedded", "workers"):
        assert f"ca13 {tag} {want}" in r.stdout, (tag, want, r.stdout)


@pytest.mark.slow
def test_full_size_r16_properties():
    """n = 2^16: λ tile, BB tile and λ per-cell kernels agree (mode equivalence at full
    size) on SW / RD / one CA step, RD equals the reference's value (App. B.2), and the
    populations are consistent."""
    torch = pytest.importorskip("torch")
    from paper_2004_13475_b200 import device as dev
    r, n = 16, 1 << 16
    s = torch.cuda.current_stream().cuda_stream
    c = cfg(r=r, rho=32)
    a = torch.zeros((n, n), dtype=torch.int64, device="cuda")
    vals = torch.from_numpy(nbb.random_member_values(GASKET, r, 17, 100)).cuda()
    dev.scatter_members_dev(c, vals.data_ptr(), a.data_ptr(), s)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    for cc in (c, cfg(r=r, rho=32, mode=MapMode.BoundingBox), cfg(r=r, rho=16),
               cfg(r=r, rho=32, kernel=KernelFamily.PerCell)):
        dev.reduction_dev(cc, a.data_ptr(), out.data_ptr(), s)
        assert int(out.item()) == 2131135664
    del vals
    # CA: seed 17 mod 2 (BASELINE C3)
    a.zero_()
    vals = torch.from_numpy(nbb.random_member_values(GASKET, r, 17, 2)).cuda()
    dev.scatter_members_dev(c, vals.data_ptr(), a.data_ptr(), s)
    pop0 = int(a.sum().item())
    assert pop0 == int(vals.sum().item())
    b = torch.zeros_like(a)
    dev.ca_step_dev(c, a.data_ptr(), b.data_ptr(), CaRule(), s)
    ref_sum = int(b.sum().item())
    rows, cols = b.sum(dim=1), b.sum(dim=0)  # checksum pair: row and column populations
    for cc in (cfg(r=r, rho=32, mode=MapMode.BoundingBox), cfg(r=r, rho=16),
               cfg(r=r, rho=32, kernel=KernelFamily.PerCell)):
        b.zero_()
        dev.ca_step_dev(cc, a.data_ptr(), b.data_ptr(), CaRule(), s)
        assert int(b.sum().item()) == ref_sum
        assert torch.equal(b.sum(dim=1), rows) and torch.equal(b.sum(dim=0), cols)
    # uint8 path agrees too
    a8 = torch.zeros((n, n), dtype=torch.uint8, device="cuda")
    b8 = torch.zeros_like(a8)
    c8 = cfg(r=r, rho=32, cell_width=1)
    dev.pack_alive_dev(c8, a.data_ptr(), a8.data_ptr(), s)
    dev.ca_step_dev(c8, a8.data_ptr(), b8.data_ptr(), CaRule(), s)
    assert int(b8.sum(dtype=torch.int64).item()) == ref_sum
    del a8, b8
    # and the 1-bit packed state: pack -> step -> unpack reproduces the int64 step exactly
    c1 = cfg(r=r, rho=32, cell_width=0)
    w1 = torch.zeros((n, n // 32), dtype=torch.int32, device="cuda")
    w2 = torch.zeros_like(w1)
    dev.pack_alive_dev(c1, a.data_ptr(), w1.data_ptr(), s)
    for cc in (c1, cfg(r=r, rho=32, cell_width=0, mode=MapMode.BoundingBox)):
        w2.zero_()
        dev.ca_step_dev(cc, w1.data_ptr(), w2.data_ptr(), CaRule(), s)
        b.zero_()
        dev.unpack_alive_dev(c1, w2.data_ptr(), b.data_ptr(), s)
        assert int(b.sum().item()) == ref_sum
        assert torch.equal(b.sum(dim=1), rows) and torch.equal(b.sum(dim=0), cols)
    # the compact (λ-ordered) state: codec -> pipelined compact step -> codec, bit-identical
    del w1, w2
    ref = torch.zeros_like(a)
    dev.ca_step_dev(c, a.data_ptr(), ref.data_ptr(), CaRule(), s)
    k1 = torch.empty(3 ** r, dtype=torch.int64, device="cuda")
    k2 = torch.empty_like(k1)
    dev.compact_store_dev(c, a.data_ptr(), k1.data_ptr(), s)
    dev.ca_compact_step_dev(c, k1.data_ptr(), k2.data_ptr(), CaRule(), s)
    dev.compact_load_dev(c, k2.data_ptr(), b.data_ptr(), 0, s)
    assert torch.equal(b, ref)
    assert int(k2.sum().item()) == ref_sum


@pytest.mark.parametrize("r", [5, 6, 7, 8, 10, 13])
def test_compact_ca_two_steps_per_pass(r):
    """ca_compact2_kernel (two steps per pass, radius-2 halo) against the oracle and against
    one launch per step (NBB_FLAG_SINGLE_STEP): random alive values (and values with other
    non-zero bit patterns) for every rule in RULES — incl. births at 0 and 8 neighbours — and
    step counts that use 0, 2 and 4 pair launches, odd and even."""
    import torch
    from paper_2004_13475_b200 import _abi as abi
    from paper_2004_13475_b200 import device as dev
    members = 3 ** r
    s = torch.cuda.current_stream().cuda_stream
    for rule in RULES:
        init = orc_random_member_grid(r, 900 + r, 2)
        for steps in (4, 5, 8, 9):
            want = orc_ca(r, init, steps, rule.birth, rule.survive)
            got = nbb.run_ca(cfg(r=r, rho=32, flags=abi.FLAG_COMPACT_STATE), grid(init, r), steps, rule)
            assert np.array_equal(got.grid.values, want), (r, rule, steps)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(r)
        x0 = torch.randint(-3, 3, (members,), dtype=torch.int64, device="cuda", generator=gen)
        outs = []
        for flags in (0, abi.FLAG_SINGLE_STEP):
            a, b = x0.clone(), torch.empty_like(x0)
            dev.ca_compact_run_dev(cfg(r=r, rho=32, flags=flags), a.data_ptr(), b.data_ptr(), 12, rule, s)
            outs.append(a)
        assert torch.equal(outs[0], outs[1]), (r, rule)


@pytest.mark.parametrize("r", [16, 17])
def test_compact_ca_two_steps_per_pass_full_size(r):
    """At full size: 8 steps as 4 pair launches equal 8 single-step launches, bit for bit."""
    import torch
    from paper_2004_13475_b200 import _abi as abi
    from paper_2004_13475_b200 import device as dev
    s = torch.cuda.current_stream().cuda_stream
    gen = torch.Generator(device="cuda")
    gen.manual_seed(4200 + r)
    x0 = torch.randint(0, 2, (3 ** r,), dtype=torch.int64, device="cuda", generator=gen)
    outs = []
    for flags in (0, abi.FLAG_SINGLE_STEP):
        a, b = x0.clone(), torch.empty_like(x0)
        dev.ca_compact_run_dev(cfg(r=r, rho=32, flags=flags), a.data_ptr(), b.data_ptr(), 8, CaRule(), s)
        outs.append(a)
        del b
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("r", [17, 18])
def test_compact_ca_full_size_sampled(r):
    """C5 size (n = 2^17, 3^17 members): two steps through the library's step loop, then a third
    step checked against the oracle rule on 600k sampled cells — uniform, every tile-corner
    cell of the first and last 2000 tiles (the halo-reading cells), and the array's ends."""
    import torch
    from paper_2004_13475_b200 import device as dev
    members = 3 ** r
    c = cfg(r=r, rho=32)
    s = torch.cuda.current_stream().cuda_stream
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1700 + r)
    a = torch.randint(0, 2, (members,), dtype=torch.int64, device="cuda", generator=gen)
    b = torch.empty_like(a)
    dev.ca_compact_run_dev(c, a.data_ptr(), b.data_ptr(), 2, CaRule(), s)  # result in a
    dev.ca_compact_step_dev(c, a.data_ptr(), b.data_ptr(), CaRule(), s)
    torch.cuda.synchronize()
    src, dst = a.cpu().numpy(), b.cpu().numpy()
    del a, b
    assert set(np.unique(dst)) <= {0, 1}
    W = 3 ** ((r + 1) // 2)
    Hb = 3 ** ((r - 5) // 2)
    rng = np.random.default_rng(r)
    tiles = np.concatenate([np.arange(2000), np.arange(3 ** (r - 5) - 2000, 3 ** (r - 5))])
    rows, cols = np.meshgrid([0, 8], [0, 26], indexing="ij")  # corner cells of the 9 x 27 block
    corner = ((tiles // Hb * 9)[:, None] + rows.ravel()[None]) * W + \
             ((tiles % Hb) * 27)[:, None] + cols.ravel()[None]
    offs = np.concatenate([rng.integers(0, members, 600_000), corner.ravel(),
                           np.arange(1000), np.arange(members - 1000, members)]).astype(np.int64)
    assert orc_ca_compact_check(r, src, dst, offs) == 0


@pytest.mark.parametrize("rho,mode", [(1, "lambda"), (4, "lambda"), (32, "lambda"), (8, "bb"), (32, "bb")])
def test_device_functor_launch(rho, mode):
    """include/nbb_launch.cuh — launch(config, kernel) with device functors: run_single_write and
    run_reduction written as functors give the oracle's grid and sum, over λ and BB launches."""
    import subprocess
    from test_capi import build_launch_example
    r, seed = 10, 31
    exe = build_launch_example("/tmp/nbb_launch_example_gpu")
    out = subprocess.run([exe, str(r), str(rho), mode, str(seed)], capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    f = out.stdout.split()
    assert f[1] == fnv1a64(orc_single_write(r))
    assert int(f[3]) == orc_reduction(r, orc_random_member_grid(r, seed, 1000))
    assert int(f[7]) == 3 ** r  # active threads = the members (closed-form counters)


@pytest.mark.parametrize("steps", [3, 4, 9])
def test_host_buffer_compact_ca_pinned_zero_copy(steps):
    """nbb_gpu_ca on pinned host Grids with FLAG_OUT_ZEROED | FLAG_COMPACT_STATE: member sectors
    read and written zero-copy (the e2e path of the bench) — bit-exact with the oracle at
    n = 2^13, twice (cached device buffers); 4 and 9 steps run two-step passes."""
    import ctypes
    import torch
    r = 13
    n = 1 << r
    g = orc_random_member_grid(r, 2024, 2)
    want = orc_ca(r, g, steps)
    hin = torch.from_numpy(g.copy()).pin_memory()
    for trial in range(2):  # the second call reuses the cached device buffers
        hout = torch.zeros((n, n), dtype=torch.int64).pin_memory()
        cc = cfg(r=r, rho=32, flags=_abi.FLAG_OUT_ZEROED | _abi.FLAG_COMPACT_STATE).to_c()
        rc = _abi.load().nbb_gpu_ca(ctypes.byref(cc), ctypes.c_void_p(hin.data_ptr()), r, steps, 8, 12,
                                    ctypes.c_void_p(hout.data_ptr()), None)
        assert rc == 0, _abi.load().nbb_gpu_last_error()
        assert np.array_equal(hout.numpy(), want), trial


@pytest.mark.parametrize("r", [5, 8, 11])
def test_ca_run_dev_embedded_temporal_blocking(r):
    """nbb_gpu_ca_run_dev on embedded int64 device grids: the gasket's run goes through the compact
    state in passes (temporal blocking of the embedded layout) — every step count equals the oracle,
    the result lands where single steps leave it, non-member cells stay 0; pass_steps, a generic rule,
    BB mode and one launch per step agree."""
    torch = pytest.importorskip("torch")
    from paper_2004_13475_b200 import device as dev
    n = 1 << r
    s = torch.cuda.current_stream().cuda_stream
    init = orc_random_member_grid(r, 90 + r, 2)
    for rule in RULES[:2]:
        for steps in (1, 2, 7, 20):
            want = orc_ca(r, init, steps, rule.birth, rule.survive)
            for kw in ({}, {"pass_steps": 3}, {"mode": MapMode.BoundingBox}, {"flags": _abi.FLAG_SINGLE_STEP}):
                a = torch.from_numpy(init.copy()).cuda()
                b = torch.zeros_like(a)
                st = dev.ca_run_dev(cfg(r=r, rho=32, **kw), a.data_ptr(), b.data_ptr(), steps, rule, s)
                assert st.result_in_b == steps % 2
                out = (b if steps % 2 else a).cpu().numpy()
                assert np.array_equal(out, want), (rule, steps, kw)
                if kw == {} and steps >= 2:
                    assert st.passes < steps  # blocked: several steps per pass
