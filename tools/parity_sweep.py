"""Randomised parity sweep (beyond the test suite): random levels, seeds, value ranges, CA rules
and step counts through every kernel family and state layout, each result compared bit for bit
with the C oracle. Prints one JSON summary line (counts per family, first mismatches if any).

    python tools/parity_sweep.py [seconds=600]
"""
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from _oracle import orc_ca, orc_random_member_grid, orc_reduction, orc_single_write  # noqa: E402
from paper_2004_13475_b200 import _abi, nbb  # noqa: E402

G = nbb.FractalSpec.sierpinski()
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 600.0
rng = random.Random(int(os.environ.get("SWEEP_SEED", "20261017")))
t_end = time.time() + budget
counts, bad = {}, []


def cfg(**kw):
    c = nbb.DispatchConfig(max_cells=1 << 28)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def check(name, ok, info):
    counts[name] = counts.get(name, 0) + 1
    if not ok and len(bad) < 20:
        bad.append({"family": name, **info})


def families(r):
    fam = []
    for mode in (nbb.MapMode.Lambda, nbb.MapMode.BoundingBox):
        for rho in (1, 2, 4, 8, 16, 32):
            if rho > (1 << r):
                continue
            fam.append((f"percell_{mode.name}_rho{rho}", cfg(r=r, rho=rho, mode=mode, kernel=nbb.KernelFamily.PerCell)))
            if mode == nbb.MapMode.Lambda and rho >= 2:
                for st in (nbb.IntraBlockStrategy.FurtherUnrolling, nbb.IntraBlockStrategy.SharedLookupTable):
                    fam.append((f"percell_lambda_rho{rho}_{st.name}",
                                cfg(r=r, rho=rho, strategy=st, kernel=nbb.KernelFamily.PerCell)))
                for be in (nbb.LambdaBackend.MmaV1, nbb.LambdaBackend.MmaV2):
                    fam.append((f"percell_lambda_rho{rho}_{be.name}",
                                cfg(r=r, rho=rho, backend=be, kernel=nbb.KernelFamily.PerCell)))
            if rho in (8, 16, 32) and r >= 5:
                fam.append((f"tile_{mode.name}_rho{rho}", cfg(r=r, rho=rho, mode=mode, kernel=nbb.KernelFamily.Tile)))
        if r >= 5:
            fam.append((f"tile_{mode.name}_u8", cfg(r=r, rho=32, mode=mode, cell_width=1, kernel=nbb.KernelFamily.Tile)))
            fam.append((f"tile_{mode.name}_bit", cfg(r=r, rho=32, mode=mode, cell_width=0, kernel=nbb.KernelFamily.Tile)))
    if r >= 5:
        fam.append(("compact_state", cfg(r=r, rho=32, flags=_abi.FLAG_COMPACT_STATE)))
        fam.append(("compact_state_bb", cfg(r=r, rho=32, mode=nbb.MapMode.BoundingBox,
                                            flags=_abi.FLAG_COMPACT_STATE)))
    return fam


def generic_families(spec, r):
    """Vicsek / carpet (s = 3): the per-cell kernels with the table-driven λ, ρ = 1, 3, 9."""
    fam = []
    for mode in (nbb.MapMode.Lambda, nbb.MapMode.BoundingBox):
        for rho in (1, 3, 9):
            if rho <= spec.side_length(r):
                fam.append((f"{spec.name}_percell_{mode.name}_rho{rho}",
                            cfg(spec=spec, r=r, rho=rho, mode=mode, kernel=nbb.KernelFamily.PerCell)))
    return fam


it = 0
while time.time() < t_end:
    it += 1
    spec = G if it % 4 else (nbb.FractalSpec.vicsek() if it % 8 else nbb.FractalSpec.carpet())
    r = rng.randint(1, 12) if spec is G else rng.randint(1, 4)
    seed = rng.randrange(1 << 30)
    modulus = rng.choice([2, 3, 100, 1 << 20, 1 << 62])
    g = orc_random_member_grid(r, seed, modulus, spec)
    rule = nbb.CaRule(birth=rng.randrange(1, 1 << 9), survive=rng.randrange(0, 1 << 9))
    steps = rng.randint(0, 6)
    want_ca = orc_ca(r, g, steps, rule.birth, rule.survive, spec)
    want_rd = orc_reduction(r, g, spec)
    want_sw = orc_single_write(r, spec)
    grid = nbb.Grid(spec, r, g)
    for name, c in (families(r) if spec is G else generic_families(spec, r)):
        info = {"spec": spec.name, "r": r, "seed": seed, "modulus": modulus, "rule": [rule.birth, rule.survive],
                "steps": steps}
        try:
            # every state layout keeps the reference's int64 Grid at the boundary
            out = nbb.run_ca(c, grid, steps, rule).grid.values
            check(name + ":ca", np.array_equal(out, want_ca), info)
            if c.cell_width == 8 and not name.startswith("compact_state"):
                check(name + ":rd", nbb.run_reduction(c, grid).value == want_rd, info)
                check(name + ":sw", np.array_equal(nbb.run_single_write(c).grid.values, want_sw), info)
        except nbb.NbbError as e:  # configurations the reference rejects are rejected here too
            check(name + ":rejected", True, {**info, "why": str(e)[:80]})

print(json.dumps({"seconds": budget, "checks": sum(counts.values()), "mismatches": len(bad),
                  "families": len(counts), "first_mismatches": bad, "counts": counts}))
