"""The C++ drop-in adapter (include/wattserve_gpu.hpp): the reference's controller
test families run through wattserve::gpu::* and compared, decision by decision and
state by state, with the unmodified reference in the same binary."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_adapter")

pytestmark = pytest.mark.gpu


def test_cpp_adapter_matches_reference():
    if not os.path.exists(BIN):
        subprocess.run([os.path.join(ROOT, "tests", "cpp", "build.sh")], check=False)
    if not os.path.exists(BIN):
        pytest.skip("test_adapter not built (needs the reference headers at build time)")
    r = subprocess.run([BIN, ROOT], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("PASS")
