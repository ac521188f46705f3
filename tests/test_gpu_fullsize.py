"""Full-size parity of the headline: C3 (n = 2^16) and C5 (n = 2^17), every cell.

BASELINE north_star: "the λ(ω) CA step on a 2^16 gasket is bit-exact with the CPU oracle".
The reference being matched is run_ca (/root/reference/proj/src/dispatch.cpp:517-557) on
random_member_grid(gasket, 16, seed 17, modulus 2) (dispatch.cpp:133-149), rule B3/S23.

Checkers (test infrastructure only):
  * the C oracle's whole-trajectory restatement on the compact state (orc_random_member_compact,
    orc_ca_compact — pinned to the dense oracle and to the reference in test_oracle.py), which
    compares all 3^16 (3^17) cells after every step count;
  * tests/golden/c3_r16.json — population + FNV-1a of the compact state after 1..20 steps, made
    by running the UNMODIFIED reference at n = 2^16 (tests/golden/make_golden_c3.py).
"""
import json
import os

import numpy as np
import pytest

from _oracle import ROOT, fnv1a64, orc_ca_compact, orc_lambda_coords, orc_random_member_compact
from paper_2004_13475_b200 import _abi, nbb
from paper_2004_13475_b200.nbb import CaRule, DispatchConfig

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLDEN = os.path.join(ROOT, "tests", "golden", "c3_r16.json")
CONWAY = CaRule()
B25S34 = CaRule(birth=(1 << 2) | (1 << 5), survive=(1 << 3) | (1 << 4))


def cfg(r, **kw):
    c = DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, device=0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def golden():
    if not os.path.exists(GOLDEN):
        return None
    with open(GOLDEN) as f:
        return json.load(f)


def run_compact(torch, r, c0, steps, rule, flags=0, pass_steps=0):
    """nbb_gpu_ca_compact_run_dev from the initial compact state; the result back on the host."""
    from paper_2004_13475_b200 import device as dev
    s = torch.cuda.current_stream().cuda_stream
    a = torch.from_numpy(c0).cuda()
    b = torch.empty_like(a)
    dev.ca_compact_run_dev(cfg(r, flags=flags, pass_steps=pass_steps), a.data_ptr(), b.data_ptr(), steps, rule, s)
    out = (a if steps % 2 == 0 else b).cpu().numpy()
    del a, b
    return out


def test_c3_initial_state_full_size():
    """The product's input path (member values in row order -> device scatter into the int64
    Grid -> compact_store_dev) gives the oracle's compact random_member_grid(16, 17, 2), which is
    the reference's (golden digest)."""
    import torch
    from paper_2004_13475_b200 import device as dev
    r, n = 16, 1 << 16
    s = torch.cuda.current_stream().cuda_stream
    c = cfg(r)
    emb = torch.zeros((n, n), dtype=torch.int64, device="cuda")
    vals = torch.from_numpy(nbb.random_member_values(nbb.FractalSpec.sierpinski(), r, 17, 2)).cuda()
    dev.scatter_members_dev(c, vals.data_ptr(), emb.data_ptr(), s)
    del vals
    comp = torch.empty(3 ** r, dtype=torch.int64, device="cuda")
    dev.compact_store_dev(c, emb.data_ptr(), comp.data_ptr(), s)
    got = comp.cpu().numpy()
    del emb, comp
    want = orc_random_member_compact(r, 17, 2)
    assert np.array_equal(got, want)
    g = golden()
    if g is not None:
        assert fnv1a64(want) == g["trajectories"]["B3/S23"]["0"]["fnv"]


@pytest.mark.parametrize("rule_name", ["B3/S23", "B25/S34"])
def test_c3_compact_trajectory_full_size(rule_name):
    """C3 at full size on the headline path (the compact state, several steps per pass): for
    every step count in (1, 2, 3, 4, 5, 8, 20) — which between them exercise every pass length the
    library issues and both result buffers — all 3^16 cells equal the oracle's trajectory, and
    the digests equal the reference's. One launch per step (NBB_FLAG_SINGLE_STEP) agrees too."""
    import torch
    rule = CONWAY if rule_name == "B3/S23" else B25S34
    r = 16
    c0 = orc_random_member_compact(r, 17, 2)
    g = golden()
    gt = g["trajectories"].get(rule_name) if g else None
    targets = (1, 2, 3, 4, 5, 8, 20) if rule_name == "B3/S23" else (1, 2, 4, 7)
    want, done = c0, 0
    for k in targets:
        want = orc_ca_compact(r, want, k - done, rule.birth, rule.survive)
        done = k
        got = run_compact(torch, r, c0, k, rule)
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, (rule_name, k, bad.size, bad[:8])
        if gt is not None and str(k) in gt:
            assert (int(want.sum()), fnv1a64(want)) == (gt[str(k)]["population"], gt[str(k)]["fnv"]), k
        if k in (4, 20):
            single = run_compact(torch, r, c0, k, rule, flags=_abi.FLAG_SINGLE_STEP)
            assert np.array_equal(single, want), (rule_name, k, "single step")


def test_c3_passes_of_12_full_size():
    """C3 at full size in passes of up to 12 steps (pass_steps = 12: the cluster kernel with the
    radius-12 halo): all 3^16 cells equal the oracle after 9, 12, 20 and 24 steps, and the
    digests equal the reference's."""
    import torch
    r = 16
    c0 = orc_random_member_compact(r, 17, 2)
    g = golden()
    gt = g["trajectories"].get("B3/S23") if g else None
    want, done = c0, 0
    for k in (9, 12, 20, 24):
        want = orc_ca_compact(r, want, k - done, CONWAY.birth, CONWAY.survive)
        done = k
        got = run_compact(torch, r, c0, k, CONWAY, pass_steps=12)
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, (k, bad.size, bad[:8])
        if gt is not None and str(k) in gt:
            assert (int(want.sum()), fnv1a64(want)) == (gt[str(k)]["population"], gt[str(k)]["fnv"]), k


def test_c3_embedded_int64_one_step_full_size():
    """The reference's own int64 embedded Grid on the device (2 x 32 GiB): one λ-tile CA step
    (ca_pipe_kernel) — every member cell equals the oracle and every non-member cell is 0."""
    import torch
    from paper_2004_13475_b200 import device as dev
    r, n = 16, 1 << 16
    s = torch.cuda.current_stream().cuda_stream
    c = cfg(r)
    c0 = orc_random_member_compact(r, 17, 2)
    xy = orc_lambda_coords(r)
    flat = torch.from_numpy(xy[:, 1] * n + xy[:, 0]).cuda()
    del xy
    a = torch.zeros(n * n, dtype=torch.int64, device="cuda")
    a[flat] = torch.from_numpy(c0).cuda()
    b = torch.zeros_like(a)
    dev.ca_step_dev(c, a.data_ptr(), b.data_ptr(), CONWAY, s)
    del a
    got = b[flat].cpu().numpy()
    total = int(b.sum().item())
    del b, flat
    want = orc_ca_compact(r, c0, 1)
    assert np.array_equal(got, want)
    assert total == int(want.sum())  # values are 0/1: no non-member cell is set


@pytest.mark.parametrize("steps", [2, 5])
def test_c5_r17_compact_all_cells(steps):
    """C5 size (n = 2^17, 3^17 = 129,140,163 cells), seed 18: every cell after 2 and 5 steps."""
    import torch
    r = 17
    c0 = orc_random_member_compact(r, 18, 2)
    got = run_compact(torch, r, c0, steps, CONWAY)
    want = orc_ca_compact(r, c0, steps)
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, (steps, bad.size, bad[:8])
