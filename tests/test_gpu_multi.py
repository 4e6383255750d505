"""N>1 GPUs: one rank per GPU over NCCL, bit-exact per-node results vs the reference.

Runs scripts/mgpu_check.py under torchrun on every visible GPU (2..8); skipped with < 2 GPUs.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
def test_multi_gpu_shuffle_matches_reference_per_node():
    n = min(_gpus(), 8)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
                        "--master-addr", "127.0.0.1", "--master-port", "29533",
                        os.path.join(ROOT, "scripts", "mgpu_check.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "FAILURES 0" in r.stdout
