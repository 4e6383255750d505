"""Engine fallbacks against the reference's golden results: the nvcc-built interpreter kernel
(k_scan; used when the NVRTC query compiler is unavailable, PSG_JIT=0 - the JIT-only
specialisations such as the owner probe, packed shuffle rows and fused NVLink path are switched
off by the engine in that mode), the hashed aggregation table at one GPU (PSG_RANK_TABLE=0) and
the row-ordered rank-table build (PSG_RANK_HOT_SEQ=0) and strided tile order (PSG_CONTIG_TILES=0)."""
import json
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


def _tables(out):
    line = [x for x in out.splitlines() if x.startswith("AGG_TABLES")][0]
    return {int(k): v for k, v in json.loads(line.split(" ", 1)[1]).items()}


def test_rank_table_on_small_cases_matches_golden():
    """PSG_SCREEN_MIN_MB=0: every one-GPU grouped join gets the membership screen, so the small
    golden cases (dense unique o_orderkey) run through the exact key bitmap and the rank-indexed
    table (k_bitmap_set, k_rank_hot, k_rank_build, the rank probe) - asserted from psg_stats."""
    env = dict(os.environ, PSG_SCREEN_MIN_MB="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "golden_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "BAD 0" in r.stdout
    assert _tables(r.stdout).get(4, 0) > 0, r.stdout[-500:]


def test_rank_records_three_launch_path_matches_golden():
    """PSG_RANK_FUSED=0: the rank records built by popcount + CUB scan + record build instead of
    the two-launch tile kernels (k_rank_tiles, k_rank_build) - the same results on the small cases."""
    env = dict(os.environ, PSG_SCREEN_MIN_MB="0", PSG_RANK_FUSED="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "golden_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "BAD 0" in r.stdout
    assert _tables(r.stdout).get(4, 0) > 0, r.stdout[-500:]


def test_bucket_overflow_list_matches_golden():
    """PSG_BUCKET_CAP=8: tiny aggregation buckets, so most matched rows go through the overflow
    list that every bucket CTA folds - results unchanged."""
    env = dict(os.environ, PSG_SCREEN_MIN_MB="0", PSG_BUCKET_CAP="8")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "golden_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "BAD 0" in r.stdout
    n = int([x for x in r.stdout.splitlines() if x.startswith("BUCKET_OVERFLOW")][0].split()[1])
    assert n > 0


def test_bucket_overflow_rerun_matches_golden():
    """PSG_BUCKET_CAP=8 + PSG_BUCKET_OVF_CAP=4: the overflow list itself overflows, so the query is
    re-run with direct table updates - results unchanged."""
    env = dict(os.environ, PSG_SCREEN_MIN_MB="0", PSG_BUCKET_CAP="8", PSG_BUCKET_OVF_CAP="4")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "golden_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "BAD 0" in r.stdout


def test_rank_table_row_ordered_build_matches_golden():
    """PSG_SCREEN_MIN_MB=0 + PSG_RANK_HOT_SEQ=0: the rank table's hot slots written by the
    row-ordered build pass (incl. its 16-byte-store branch) on the small golden cases."""
    env = dict(os.environ, PSG_SCREEN_MIN_MB="0", PSG_RANK_HOT_SEQ="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "golden_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "BAD 0" in r.stdout
    assert _tables(r.stdout).get(4, 0) > 0, r.stdout[-500:]


def test_interpreter_with_screen_falls_back_to_hashed_table():
    """PSG_JIT=0 + PSG_SCREEN_MIN_MB=0: the interpreter kernel cannot run the rank-indexed table, so
    the engine must pick the hashed table (+ exact key bitmap) instead (no rank mode without JIT)."""
    env = dict(os.environ, PSG_JIT="0", PSG_SCREEN_MIN_MB="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "golden_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "BAD 0" in r.stdout
    t = _tables(r.stdout)
    assert t.get(4, 0) == 0 and t.get(3, 0) > 0, t


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


def test_peer_slab_path_on_one_gpu_matches_golden():
    """PSG_SLAB_FAKE=1: the N>1 peer-slab data path on one GPU - the probe kernel treats half the
    keys as another rank's (packed into the outbox in warp-claimed chunks, padding sentinels) and
    the owner-side fold (k_slab_consume) adds them back - so the multi-GPU kernels are
    parity-tested even on a single-GPU box; asserted to have run from psg_stats.shuffle_fused."""
    env = dict(os.environ, PSG_SCREEN_MIN_MB="0", PSG_SLAB_FAKE="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "golden_check.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "BAD 0" in r.stdout
    n = int([x for x in r.stdout.splitlines() if x.startswith("SLAB_FUSED")][0].split()[1])
    assert n > 0, r.stdout[-500:]
