"""The cluster walk of the compact CA pass (compact_cluster.cuh: batches = level-3 sub-gaskets of
27 tiles, in-cluster halo words as compile-time bit permutations) against the C oracle and
against the 32-ordinal sliced walk (NBB_PASS_IMPL=sliced), for every pass length 1..12, both rule
instantiations, levels where the orthotope holds 1, 3 and 81 cluster columns."""
import os

import numpy as np
import pytest

from _oracle import orc_ca_compact, orc_random_member_compact
from paper_2004_13475_b200.nbb import CaRule, DispatchConfig

pytestmark = pytest.mark.gpu

HIGHLIFE = CaRule(birth=(1 << 3) | (1 << 6), survive=(1 << 2) | (1 << 3))


def run(torch, r, c0, steps, rule, k, impl):
    from paper_2004_13475_b200 import device as dev
    old = os.environ.get("NBB_PASS_IMPL")
    os.environ["NBB_PASS_IMPL"] = impl
    try:
        s = torch.cuda.current_stream().cuda_stream
        a = torch.from_numpy(c0).cuda()
        b = torch.empty_like(a)
        c = DispatchConfig(r=r, rho=32, max_cells=(1 << r) ** 2, device=0, pass_steps=k)
        st = dev.ca_compact_passes_dev(c, a.data_ptr(), b.data_ptr(), steps, rule, s)
        return (b if st.result_in_b else a).cpu().numpy()
    finally:
        if old is None:
            del os.environ["NBB_PASS_IMPL"]
        else:
            os.environ["NBB_PASS_IMPL"] = old


@pytest.mark.parametrize("r", [8, 10, 13])
@pytest.mark.parametrize("rule", [CaRule(), HIGHLIFE], ids=["B3S23", "B36S23"])
def test_cluster_walk_matches_oracle_every_pass_length(r, rule):
    torch = pytest.importorskip("torch")
    c0 = orc_random_member_compact(r, 40 + r, 2)
    steps = 25
    want = orc_ca_compact(r, c0, steps, rule.birth, rule.survive)
    for k in range(1, 13):
        got = run(torch, r, c0, steps, rule, k, "cluster")
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, (r, k, bad.size, bad[:8])
    # the sliced walk (passes of <= 8) gives the same state
    assert np.array_equal(run(torch, r, c0, steps, rule, 8, "sliced"), want)


def test_cluster_walk_arbitrary_int64_values():
    """Alive means != 0 for any int64 in the initial state (values with only the high word set,
    negative values): the loader folds both halves."""
    torch = pytest.importorskip("torch")
    r = 11
    rng = np.random.default_rng(7)
    c0 = orc_random_member_compact(r, 3, 2)
    raw = np.where(c0 != 0, rng.choice(np.array([1, -1, 1 << 32, -(1 << 40), 7], dtype=np.int64),
                                       size=c0.shape), 0).astype(np.int64)
    want = orc_ca_compact(r, c0, 12, CaRule().birth, CaRule().survive)
    for k in (1, 8, 12):
        assert np.array_equal(run(torch, r, raw, 12, CaRule(), k, "cluster"), want), k


def test_cluster_walk_random_rules():
    """Runtime rules (RuleTab: the rule as mux-tree constants in the kernel parameters) for 40
    random birth / survive masks over counts 0..8, including count-0 births and count-8 survival,
    in passes of 8 and 12 steps, against the oracle."""
    torch = pytest.importorskip("torch")
    r = 10
    rng = np.random.default_rng(2026)
    c0 = orc_random_member_compact(r, 77, 2)
    rules = [CaRule(birth=int(b), survive=int(s)) for b, s in rng.integers(0, 1 << 9, size=(38, 2))]
    rules += [CaRule(birth=1 | (1 << 8), survive=1 << 8), CaRule(birth=0x1FF, survive=0)]
    for rule in rules:
        want = orc_ca_compact(r, c0, 13, rule.birth, rule.survive)
        for k in (8, 12):
            got = run(torch, r, c0, 13, rule, k, "cluster")
            assert np.array_equal(got, want), (rule.birth, rule.survive, k)
        assert np.array_equal(run(torch, r, c0, 13, rule, 8, "sliced"), want), (rule.birth, rule.survive)
