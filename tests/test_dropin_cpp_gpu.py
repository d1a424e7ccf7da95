"""GPU: the C++ drop-in (include/shardplan_gpu.hpp) against the unmodified
reference library, call for call (tests/cpp/test_dropin.cpp)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "test_dropin")


@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in test binary not built (needs reference headers)")
def test_cpp_dropin_matches_reference(cuda_ctx):
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout
