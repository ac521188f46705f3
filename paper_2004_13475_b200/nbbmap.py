"""`nbbmap bench` over the GPU path — the reference CLI's reporting contract
(tools/nbbmap.cpp:530-625) with the same options, seeds and CSV bytes:

    python -m paper_2004_13475_b200.nbbmap bench --workload ca --rmin 2 --rmax 6 \\
        --rho 1,2,4 --mode both --seed 7 [--timing] [--out file.csv]

Rows are WorkReport.csv_row() + ",<workload>,<quotient>" with quotient = n^2 / threads
(C++ ostream default formatting); counters are the reference's (closed form), so with
--timing off the CSV is byte-identical to the reference's for any worker/device count.
With --timing, `micros` is the CUDA-event time of the launch (mean over --reps; for ca
the mean over the steps of one run). Exit codes follow nbbmap.cpp:747-759 (2: bad
arguments / invalid config, 3: resource limit or CUDA failure).
"""
from __future__ import annotations

import argparse
import sys

from . import nbb


def _fmt_double(q: float) -> str:
    """std::ostream << double with the default precision (6 significant, %g)."""
    return "%g" % q


def embedded_cells(spec: nbb.FractalSpec, r: int) -> int:   # nbbmap.cpp:58-64
    n = spec.s ** r
    return (1 << 64) - 1 if n > (1 << 31) else n * n


def require_cells(spec, r, max_cells):                        # nbbmap.cpp:66-73
    cells = embedded_cells(spec, r)
    if cells > max_cells:
        raise nbb.ResourceError(f"r={r} needs {cells} embedded cells, above the --max-cells "
                                f"budget of {max_cells}")


def cmd_bench(a, out, err) -> int:                            # nbbmap.cpp:530-625
    spec = nbb.FractalSpec.builtin(a.spec)
    if a.rmin > a.rmax:
        raise nbb.InvalidArgument("empty scale range: rmin > rmax")
    modes = []
    if a.mode in ("bb", "both"):
        modes.append(nbb.MapMode.BoundingBox)
    if a.mode in ("lambda", "both"):
        modes.append(nbb.MapMode.Lambda)
    out.write(nbb.WorkReport.csv_header() + ",workload,quotient\n")
    for r in range(a.rmin, a.rmax + 1):
        require_cells(spec, r, a.max_cells)
        rd_grid = ca_grid = None
        if a.workload == "rd":
            rd_grid = nbb.random_member_grid(spec, r, a.seed + r, 100, a.max_cells)
        elif a.workload == "ca":
            ca_grid = nbb.random_member_grid(spec, r, a.seed + r, 2, a.max_cells)
        for rho in a.rho:
            for mode in modes:
                cfg = nbb.DispatchConfig(
                    spec=spec, r=r, rho=rho, mode=mode, strategy=nbb.strategy_from_string(a.strategy),
                    backend=(nbb.LambdaBackend.Direct if mode == nbb.MapMode.BoundingBox
                             else nbb.backend_from_string(a.backend)),
                    workers=a.workers, timing=a.timing, max_cells=a.max_cells, device=a.device)
                try:
                    cfg.validate()
                except nbb.InvalidArgument as e:
                    err.write(f"skip r={r} rho={rho} mode={nbb.to_string(mode)}: {e}\n")
                    continue

                def run_once():
                    if a.workload == "sw":
                        return nbb.run_single_write(cfg).report
                    if a.workload == "rd":
                        return nbb.run_reduction(cfg, rd_grid).report
                    res = nbb.run_ca(cfg, ca_grid, a.steps)
                    first = res.reports[0]
                    first.micros = sum(x.micros for x in res.reports) // len(res.reports)
                    return first

                row = run_once()
                total = row.micros
                for _ in range(1, a.reps):
                    total += run_once().micros
                row.micros = total // a.reps
                q = embedded_cells(spec, r) / row.threads_launched
                out.write(f"{row.csv_row()},{a.workload},{_fmt_double(q)}\n")
    out.flush()
    return 0


def _rho_list(s: str):
    return [int(x) for x in s.split(",") if x]


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="nbbmap", description="block-space thread maps (B200 path)")
    sub = p.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="sweep launches and emit CSV")
    b.add_argument("--spec", default="sierpinski")
    b.add_argument("--workload", default="sw", choices=["sw", "rd", "ca"])
    b.add_argument("--rmin", type=int, default=0)
    b.add_argument("--rmax", type=int, default=6)
    b.add_argument("--rho", type=_rho_list, default=[1])
    b.add_argument("--mode", default="both", choices=["bb", "lambda", "both"])
    b.add_argument("--strategy", default="subbox", choices=["unroll", "lut", "subbox"])
    b.add_argument("--backend", default="direct", choices=["direct", "mma1", "mma2", "mma3"])
    b.add_argument("--reps", type=int, default=1)
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--out", default="-")
    b.add_argument("--workers", type=int, default=1)
    b.add_argument("--timing", action="store_true")
    b.add_argument("--steps", type=int, default=4)
    b.add_argument("--max-cells", dest="max_cells", type=int, default=1 << 24)
    b.add_argument("--device", type=int, default=0)
    try:
        a = p.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    if a.rmin < 0 or a.rmax < 0 or a.reps < 1 or a.workers < 1 or a.steps < 1:
        sys.stderr.write("error: option out of range\n")
        return 2
    try:
        out = sys.stdout if a.out == "-" else open(a.out, "w")
        try:
            return cmd_bench(a, out, sys.stderr)
        finally:
            if out is not sys.stdout:
                out.close()
    except (nbb.ResourceError, nbb.CudaError, MemoryError) as e:
        sys.stderr.write(f"resource limit: {e}\n")
        return 3
    except (nbb.InvalidArgument, nbb.OutOfRange, nbb.DomainError, ValueError) as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
    except RuntimeError as e:
        sys.stderr.write(f"error: {e}\n")
        return 3


if __name__ == "__main__":
    sys.exit(main())
