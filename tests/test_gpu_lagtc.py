"""The tensor-core phase-lag kernel (pairs_lagtc.cu, opt-in CSCONN_K3=tc) against
the same parity suite as the default CUDA-core kernel.

The library reads CSCONN_K3 once per process, so the parity tests of
test_gpu_parity.py that exercise the phase-lag family (golden cases, tile-boundary
shapes, exact zero-lag zeros, float32 input) are re-run in a child process with the
variant selected.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent


def test_tensor_core_k3_matches_reference():
    env = dict(os.environ, CSCONN_K3="tc")
    sel = "lag or pli_only or wpli_only or imag_pli or tile_boundary or zero_lag or float32"
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        str(HERE / "test_gpu_parity.py"), "-k", sel],
                       cwd=HERE.parent, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
