"""The nvcc-built interpreter kernel (k_scan; used when the NVRTC query compiler is unavailable,
PSG_JIT=0) against the reference's golden results. The JIT-only specialisations (owner probe,
packed shuffle rows, fused NVLink path) are switched off by the engine in that mode."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_interpreter_kernels_match_golden():
    env = dict(os.environ, PSG_JIT="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "golden_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "BAD 0" in r.stdout
