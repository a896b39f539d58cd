"""The reference-side "cuda" TransportBackend plugin (integration/cuda_backend.cpp), compiled
against the reference's own headers and library, driven through the reference's
TransportBackend contract by a C++ test binary (integration/test_cuda_backend.cpp, in the
style of proj/tests/test_backends.cpp:262-300): capabilities, metadata attach through the
reference SegmentRegistry, bit-exact copies over three media pairs, backpressure (prefix
accept), capability mismatch, fatal latch, and plugin mode end to end (the reference
SliceScheduler plans config 1, the B200 moves the bytes)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "test_cuda_backend")


def test_reference_side_cuda_backend_plugin_contract():
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/test_cuda_backend not built (needs the reference headers)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    assert "0 failed" in r.stdout
