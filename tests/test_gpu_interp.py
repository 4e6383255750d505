"""Engine fallbacks against the reference's golden results: the nvcc-built interpreter kernel
(k_scan; used when the NVRTC query compiler is unavailable, PSG_JIT=0 - the JIT-only
specialisations such as the owner probe, packed shuffle rows and fused NVLink path are switched
off by the engine in that mode), the hashed aggregation table at one GPU (PSG_RANK_TABLE=0) and
the row-ordered rank-table build (PSG_RANK_HOT_SEQ=0) and strided tile order (PSG_CONTIG_TILES=0)."""
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


def test_hashed_aggregation_table_matches_golden():
    """PSG_RANK_TABLE=0: the one-GPU grouped join uses the hashed open-addressing aggregation table
    (CAS insert) instead of the rank-indexed one; both must give the reference's results."""
    env = dict(os.environ, PSG_RANK_TABLE="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "golden_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "BAD 0" in r.stdout


def test_row_ordered_rank_build_matches_golden():
    """PSG_RANK_HOT_SEQ=0: the rank-indexed table's hot slots are written by the row-ordered build
    pass instead of k_rank_hot's slot-ordered walk of the key bitmap."""
    env = dict(os.environ, PSG_RANK_HOT_SEQ="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "golden_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "BAD 0" in r.stdout


def test_strided_tile_order_matches_golden():
    """PSG_CONTIG_TILES=0: the warp-staged compaction programs walk tiles a grid apart instead of
    one contiguous tile range per CTA."""
    env = dict(os.environ, PSG_CONTIG_TILES="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "golden_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "BAD 0" in r.stdout
