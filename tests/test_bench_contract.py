"""bench.py's reference arm (CPU): the unmodified reference's run_ca (oracle/_ref/libnbbref.so) on an
input from the C oracle, one JSON line with the contract's keys — and the product library is never
loaded on that path (the driver checks which .so files the reference arm maps)."""
import json
import os
import subprocess
import sys

import pytest

from _oracle import ROOT, REF_PATH


@pytest.mark.skipif(not os.path.exists(REF_PATH), reason="oracle/_ref/libnbbref.so not built")
def test_reference_arm_line_and_no_product_library():
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--level', '9', '--steps', '2'];"
            "runpy.run_path('bench.py', run_name='__main__');"
            "maps = open('/proc/self/maps').read();"
            "print('MAPS', int('libnbbgpu' in maps), int('libnbbref' in maps))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and "unavailable" not in line, line
    for key in ("metric", "value", "unit", "steps", "ms_per_step", "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["unit"] == "cells/s" and line["value"] > 0 and line["steps"] == 2
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert lines[-1] == "MAPS 0 1"  # the reference was loaded, the product library was not
