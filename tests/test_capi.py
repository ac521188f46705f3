"""The product C ABI without a GPU: the library loads, exports every symbol
include/nbb_gpu.h declares, its host logic (validation, counters, CSV, seeded grids)
matches the reference's, and compute entry points fail loudly (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from _oracle import GASKET, ROOT, fnv1a64
from paper_2004_13475_b200 import _abi
from paper_2004_13475_b200 import nbb
from paper_2004_13475_b200.nbb import (DispatchConfig, FractalSpec, IntraBlockStrategy,
                                       InvalidArgument, LambdaBackend, MapMode)

HEADER = os.path.join(ROOT, "include", "nbb_gpu.h")


def _cfg(**kw):
    c = DispatchConfig()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nbb_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    names = declared_symbols()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), name
        assert name in _abi.SIGNATURES, f"{name} missing from _abi.SIGNATURES"
    assert lib.nbb_gpu_abi_version() == 4


@pytest.mark.parametrize("kmax", [1, 2, 3, 4, 5, 8, 12])
def test_pass_plan(kmax):
    """nbb_gpu_pass_plan (host only): the passes a compact CA run issues — every step counted once,
    at most pass_steps per pass, the fewest passes (ceil(steps / K)) without parity; with parity
    the pass count has the parity of `steps` (result where single steps leave it), one more pass
    at most."""
    from paper_2004_13475_b200 import device as dev
    c = _cfg(r=10, rho=32, pass_steps=kmax)
    for steps in range(0, 41):
        for parity in (False, True):
            st = dev.pass_plan(c, steps, parity)
            by = list(st.by_steps)
            assert sum(k * by[k] for k in range(13)) == steps
            assert all(by[k] == 0 for k in range(kmax + 1, 13))
            assert st.passes == sum(by)
            fewest = -(-steps // kmax)
            if parity:
                assert st.passes in (fewest, fewest + 1) and st.passes % 2 == steps % 2
            else:
                assert st.passes == fewest
            assert st.result_in_b == st.passes % 2
    single = dev.pass_plan(_cfg(r=10, rho=32, flags=_abi.FLAG_SINGLE_STEP), 7)
    assert single.passes == 7 and single.by_steps[1] == 7
    with pytest.raises(nbb.InvalidArgument):
        dev.pass_plan(_cfg(r=10, rho=32, pass_steps=13), 4)
    # default 8 steps per pass; up to 12 on the cluster walk (r >= 8), 8 on the sliced walk
    assert dev.pass_plan(_cfg(r=10, rho=32), 24).passes == 3
    assert dev.pass_plan(_cfg(r=10, rho=32, pass_steps=12), 24).passes == 2
    assert dev.pass_plan(_cfg(r=7, rho=32, pass_steps=12), 24).passes == 3


def test_library_is_sm100a_and_native():
    """The .so carries sm_100a SASS (cuobjdump) — no PTX-JIT-only or CPU build."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _abi.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_config_init_defaults():
    lib = _abi.load()
    c = _abi.NbbConfig()
    lib.nbb_config_init(ctypes.byref(c))
    assert (c.spec.name, c.spec.k, c.spec.s) == (b"sierpinski", 3, 2)
    assert (c.r, c.rho, c.mode, c.strategy, c.backend, c.workers, c.cell_width) == \
        (0, 1, _abi.MODE_LAMBDA, _abi.STRATEGY_SUBBOX, _abi.BACKEND_DIRECT, 1, 8)
    assert c.max_cells == 1 << 24


def test_validation_matches_reference(golden):
    for v in golden["validation"]:
        spec = FractalSpec.builtin(v.get("spec", "sierpinski"))
        c = _cfg(spec=spec, r=v["r"], rho=v["rho"], mode=MapMode(v["mode"]),
                 strategy=IntraBlockStrategy(v["strategy"]), backend=LambdaBackend(v["backend"]),
                 workers=v["workers"])
        if v["rc"] == 0:
            c.validate()
        else:
            with pytest.raises(InvalidArgument) as e:
                c.validate()
            assert str(e.value) == v["msg"]


def test_counters_and_csv_match_reference(golden):
    for row in golden["csv_rows"]:
        c = _cfg(r=row["r"], rho=row["rho"], mode=MapMode(row["mode"]),
                 strategy=IntraBlockStrategy(row["strategy"]), backend=LambdaBackend(row["backend"]))
        rep = nbb.plan_report(c)
        assert rep.csv_row() == row["csv"]
        assert rep.map_levels == row["map_levels"]
        assert nbb.launch_block_count(c) == rep.blocks_launched


def test_csv_frozen_rows():
    """test_dispatch.cpp:344-362 and test_cli.cpp:151-156."""
    assert nbb.WorkReport.csv_header() == \
        "# spec,r,rho,mode,strategy,backend,blocks,threads,active,wasted,map_ops,micros"
    assert nbb.plan_report(_cfg(r=4, mode=MapMode.BoundingBox)).csv_row() == \
        "sierpinski,4,1,bb,subbox,direct,256,256,81,175,256,0"
    assert nbb.plan_report(_cfg(r=4)).csv_row() == "sierpinski,4,1,lambda,subbox,direct,81,81,81,0,405,0"
    lut = nbb.plan_report(_cfg(r=4, rho=4, strategy=IntraBlockStrategy.SharedLookupTable))
    assert lut.map_ops == 9 * 2 + 9 * 2 and lut.map_levels == 2
    assert nbb.plan_report(_cfg(r=8, mode=MapMode.BoundingBox)).csv_row() == \
        "sierpinski,8,1,bb,subbox,direct,65536,65536,6561,58975,65536,0"
    assert nbb.plan_report(_cfg(r=8)).csv_row() == \
        "sierpinski,8,1,lambda,subbox,direct,6561,6561,6561,0,59049,0"
    v2 = nbb.plan_report(_cfg(r=4, rho=2, backend=LambdaBackend.MmaV2))
    assert (v2.blocks_launched, v2.threads_launched, v2.threads_active, v2.threads_wasted) == \
        (100, 100, 81, 19)


def test_work_quotient():
    bb8 = nbb.plan_report(_cfg(r=8, mode=MapMode.BoundingBox))
    lam8 = nbb.plan_report(_cfg(r=8))
    assert nbb.work_quotient(bb8, lam8) == pytest.approx(65536 / 6561)
    assert nbb.work_quotient(bb8, lam8, True) == pytest.approx(65536 / 6561 / 8)
    with pytest.raises(InvalidArgument):
        nbb.work_quotient(lam8, bb8)
    with pytest.raises(InvalidArgument):
        nbb.work_quotient(bb8, nbb.plan_report(_cfg(r=6)))
    bb0, lam0 = nbb.plan_report(_cfg(r=0, mode=MapMode.BoundingBox)), nbb.plan_report(_cfg(r=0))
    assert nbb.work_quotient(bb0, lam0) == 1.0 and nbb.work_quotient(bb0, lam0, True) == 1.0


def test_random_member_grid_matches_reference(golden):
    for r in range(0, 13):
        w = golden["workloads"][str(r)]
        g = nbb.random_member_grid(GASKET, r, 1 + r, 100)
        assert fnv1a64(g.values) == w["rd_grid_fnv"]
        v = nbb.random_member_values(GASKET, r, 1 + r, 100)
        n = 1 << r
        yy, xx = np.mgrid[0:n, 0:n]
        assert np.array_equal(g.values[(xx & (n - 1 - yy)) == 0], v)
    with pytest.raises(InvalidArgument):
        nbb.random_member_grid(GASKET, 3, 1, 0)
    with pytest.raises(nbb.ResourceError):
        nbb.random_member_grid(GASKET, 13, 1, 2)  # 2^26 cells > default 2^24 budget


def test_string_conversions():
    for s in ("bb", "lambda"):
        assert nbb.to_string(nbb.mode_from_string(s)) == s
    for s in ("unroll", "lut", "subbox"):
        assert nbb.to_string(nbb.strategy_from_string(s)) == s
    for s in ("direct", "mma1", "mma2", "mma3"):
        assert nbb.to_string(nbb.backend_from_string(s)) == s
    with pytest.raises(InvalidArgument):
        nbb.strategy_from_string("fu")


@pytest.mark.skipif(nbb.device_count() > 0, reason="a GPU is present")
def test_compute_fails_loudly_without_gpu():
    """No CPU fallback: every compute entry point reports NBB_ERR_CUDA."""
    c = _cfg(r=4, rho=4)
    with pytest.raises(nbb.CudaError):
        nbb.run_single_write(c)
    with pytest.raises(nbb.CudaError):
        nbb.run_reduction(c, nbb.Grid(GASKET, 4))
    with pytest.raises(nbb.CudaError):
        nbb.run_ca(c, nbb.Grid(GASKET, 4), 1)
    with pytest.raises(nbb.CudaError):
        nbb.lambda_coords(c, 3)


def test_invalid_config_rejected_before_device():
    with pytest.raises(InvalidArgument, match="rho 3 is not one of"):
        nbb.run_single_write(_cfg(r=4, rho=3))
    with pytest.raises(InvalidArgument, match="does not match the configured"):
        nbb.run_reduction(_cfg(r=3), nbb.Grid(GASKET, 2))
    with pytest.raises(InvalidArgument, match="negative step count"):
        nbb.run_ca(_cfg(r=2), nbb.Grid(GASKET, 2), -1)
    bad = FractalSpec("bad", 10, 3, tuple((i % 3, i // 3 % 3) for i in range(10)))
    with pytest.raises(InvalidArgument, match="more replicas than step-box cells"):
        nbb.run_single_write(_cfg(spec=bad, r=2))
    dup = FractalSpec("dup", 2, 2, ((0, 0), (0, 0)))
    with pytest.raises(InvalidArgument, match="overlap"):
        nbb.run_single_write(_cfg(spec=dup, r=2))
    with pytest.raises(InvalidArgument, match="1-bit CA states run on the sierpinski gasket only"):
        nbb.run_ca(_cfg(spec=FractalSpec.vicsek(), r=2, cell_width=1),
                   nbb.Grid(FractalSpec.vicsek(), 2), 1)


def test_cpp_shim_compiles():
    """include/nbb_gpu.hpp (the reference-signature C++ shim) builds against the C ABI."""
    src = os.path.join(ROOT, "tests", "cpp", "shim_example.cpp")
    out = "/tmp/nbb_shim_example"
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-Wall", "-Wextra", "-Werror",
                    f"-I{os.path.join(ROOT, 'include')}", src, "-o", out,
                    f"-L{os.path.dirname(_abi.LIB_PATH)}", "-lnbbgpu",
                    f"-Wl,-rpath,{os.path.dirname(_abi.LIB_PATH)}"], check=True)
    # without a GPU the example must fail loudly (exit 3 = CUDA error via exception)
    r = subprocess.run([out, "--host-only"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "sierpinski,8,1,lambda,subbox,direct,6561,6561,6561,0,59049,0" in r.stdout


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors (_abi.py) have the header's sizes and field offsets (gcc -> offsetof)."""
    structs = {"nbb_spec": _abi.NbbSpec, "nbb_config": _abi.NbbConfig, "nbb_report": _abi.NbbReport,
               "nbb_p2p": _abi.NbbP2P}
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "nbb_gpu.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f in py._fields_:
            lines.append(f'printf("{cname} {f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["/usr/bin/gcc", "-std=c11", f"-I{os.path.join(ROOT, 'include')}", str(src), "-o", str(exe)],
                   check=True)
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        c, f, v = line.split()
        got[(c, f)] = int(v)
    for cname, py in structs.items():
        assert got[(cname, "sizeof")] == ctypes.sizeof(py), cname
        for f in py._fields_:
            assert got[(cname, f[0])] == getattr(py, f[0]).offset, (cname, f[0])


def build_launch_example(out="/tmp/nbb_launch_example"):
    """tests/cuda/launch_example.cu: include/nbb_launch.cuh (the reference's launch(config,
    kernel) for device functors) compiled by nvcc into the caller's own binary."""
    src = os.path.join(ROOT, "tests", "cuda", "launch_example.cu")
    lib_dir = os.path.dirname(_abi.LIB_PATH)
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
                    "-std=c++17", f"-I{os.path.join(ROOT, 'include')}", src, "-o", out,
                    f"-L{lib_dir}", "-lnbbgpu", "-Xlinker", "-rpath", "-Xlinker", lib_dir], check=True)
    return out


def test_device_functor_launch_compiles_and_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present: the launch succeeds (the -m gpu tests run it)")
    exe = build_launch_example()
    r = subprocess.run([exe, "--host-only"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_nbbmap_quotient_format_matches_cpp():
    """nbbmap prints the quotient with std::ostream defaults (%g, 6 significant)."""
    from _oracle import ref_available, ref_lib
    from paper_2004_13475_b200.nbbmap import _fmt_double
    if not ref_available():
        pytest.skip("reference library not built")
    buf = ctypes.create_string_buffer(64)
    for r in range(0, 24):
        for rho in (1, 2, 4, 8, 16, 32):
            for q in (4 ** r / 3 ** r, 4 ** r / (rho * rho * 3 ** max(r - 1, 0)), 1.0, 100.0 / 81.0):
                assert ref_lib().ref_format_double(q, buf, 64) == 0
                assert _fmt_double(q) == buf.value.decode(), q


def test_nbbmap_cli_errors():
    from paper_2004_13475_b200 import nbbmap
    assert nbbmap.main(["bench", "--workload", "xx"]) == 2
    assert nbbmap.main(["bench", "--rmin", "3", "--rmax", "2"]) == 2
    assert nbbmap.main(["bench", "--rmin", "13", "--rmax", "13"]) == 3


def test_nbbc_file_matches_reference(tmp_path):
    """NBBC compact files (block_map.cpp:284-362): our writer's bytes equal the reference
    writer's, each reader reads the other's files, and the error texts match."""
    from _oracle import ref_available, ref_lib
    rng = np.random.default_rng(1)
    for spec, level in ((GASKET, 5), (FractalSpec.vicsek(), 3), (FractalSpec.carpet(), 2)):
        w, h = spec.orthotope_dims(level)
        g = nbb.CompactGrid(spec, level, rng.integers(-2**62, 2**62, size=(h, w)))
        ours = tmp_path / f"ours_{spec.name}.nbbc"
        nbb.write_compact(str(ours), spec, g)
        raw = ours.read_bytes()
        assert raw[:4] == b"NBBC" and len(raw) == 16 + 8 * w * h
        assert nbb.read_compact(str(ours), spec) == g
        if ref_available():
            theirs = tmp_path / f"ref_{spec.name}.nbbc"
            assert ref_lib().ref_write_compact(ctypes.byref(spec.to_c()), level,
                                               g.values.ctypes.data_as(ctypes.c_void_p),
                                               str(theirs).encode()) == 0
            assert theirs.read_bytes() == raw
    bad = tmp_path / "bad.nbbc"
    bad.write_bytes(b"NBBX" + bytes(12))
    with pytest.raises(InvalidArgument, match="compact file: bad magic"):
        nbb.read_compact(str(bad), GASKET)
    bad.write_bytes(raw[:20])  # carpet header, truncated payload, read as carpet
    with pytest.raises(InvalidArgument, match="truncated payload"):
        nbb.read_compact(str(bad), FractalSpec.carpet())
    with pytest.raises(InvalidArgument, match=r"header \(k=8, s=3\) does not match spec 'sierpinski'"):
        nbb.read_compact(str(ours), GASKET)
