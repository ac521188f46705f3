import json
import os
import sys

import pytest

TESTS = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(TESTS)
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running (full-size) check")
    # build (no-op when up to date): product library + test-only checkers
    from paper_2004_13475_b200 import _build
    _build.build_library()
    _build.build_oracle()


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(TESTS, "golden", "golden.json")) as f:
        return json.load(f)
