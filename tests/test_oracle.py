"""The oracle is pinned before it is trusted (CPU only).

* oracle generator (oracle/gen_oracle.c) == reference generator, byte for byte (sha256 fixtures
  made from the reference itself by tests/golden/make_golden.py);
* oracle executor (oracle/plan_oracle.py) == reference execute_plan results for every golden case,
  and == SURVEY.md §8(c)'s golden table.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from oracle import plan_oracle as po

SURVEY_GOLDEN = {  # scale -> (groups, Σrows, Σsum_price, Σsum_disc, rowhash)
    0.01: (1145, 2832, 398822051, 14207, "9c96e282d54a8f49"),
    0.1: (12080, 29797, 4177141598, 148760, "674f0fb4d84299e9"),
}


@pytest.mark.parametrize("idx", range(7))
def test_generator_bytes_match_reference(idx, gen_hashes, tmp_path):
    spec = gen_hashes[idx]
    d = str(tmp_path / "g")
    oracle.gen_tpch(d, spec["scale"], spec["nodes"], spec["devices"], spec["seed"], spec["codec"], spec["rg_bytes"])
    got = {}
    for root, _dirs, files in os.walk(d):
        for f in files:
            p = os.path.join(root, f)
            got[os.path.relpath(p, d)] = hashlib.sha256(open(p, "rb").read()).hexdigest()
    assert got == spec["files"]


def _cases(golden, max_scale=0.1):
    seen = set()
    for r in golden["results"]:
        if r["scale"] <= max_scale and r["case"] not in seen:
            seen.add(r["case"])
            yield r


def test_oracle_matches_every_reference_case(golden, datasets):
    n = 0
    for r in _cases(golden):
        d = datasets(r["scale"], r["nodes"], r["devices"], r["seed"], r["codec"], r["rg_bytes"])
        res = po.execute(json.dumps(golden["plans"][r["plan"]]), d, r["nodes"])
        s = po.summary(res)
        assert s["rows"] == r["rows"], r["case"]
        assert s["rowhash"] == r["rowhash"], r["case"]
        assert s["colsums"] == r["colsums"], r["case"]
        assert s["per_node_rows"] == r["per_node_rows"], r["case"]
        n += 1
    assert n >= 15


@pytest.mark.parametrize("scale", [0.01, 0.1])
def test_oracle_matches_survey_table(scale, golden, datasets):
    d = datasets(scale, 1, 1)
    s = po.summary(po.execute(json.dumps(golden["plans"]["canonical"]), d, 1))
    g = SURVEY_GOLDEN[scale]
    assert (s["rows"], int(s["colsums"][1]), int(s["colsums"][2]), int(s["colsums"][3]), s["rowhash"]) == g


def test_oracle_rows_match_reference_dump(golden, datasets):
    raw = np.fromfile(os.path.join(os.path.dirname(__file__), "golden", "q3_s001_rows.bin"), dtype="<u8")
    n, k = int(raw[0]), int(raw[1])
    want = raw[2:].reshape(n, k)
    d = datasets(0.01, 1, 1)
    (_schema, rows), = po.execute(json.dumps(golden["plans"]["canonical"]), d, 1)
    assert np.array_equal(rows, want)  # same rows, same (key) order


def test_partition_of_matches_reference_hash():
    keys = np.array([0, 1, 2, 3, -1, 2**62, -(2**63)], dtype=np.int64)
    with np.errstate(over="ignore"):
        for n in (1, 2, 3, 8):
            got = po.partition_of(keys.view(np.uint64), n)
            want = [(((int(k) % 2**64) * 0x9E3779B97F4A7C15 % 2**64) >> 13) % n for k in keys]
            assert list(got) == want


def test_partition_of_is_periodic_for_power_of_two_nodes():
    """The invariant k_own_table / k_or_own rely on (kernels.cu): at power-of-two n the owner of
    key k depends on k mod 2^(13 + log2 n) only, so the owned-bit mask of bitmap word w (keys
    kmin + 64 w + b) is the mask of word w mod 128 n."""
    rng = np.random.default_rng(7)
    with np.errstate(over="ignore"):
        for n in (2, 4, 8, 16):
            period = 128 * n
            for kmin in (0, -5, int(rng.integers(-(2**40), 2**40))):
                ws = rng.integers(0, 10**7, size=32)
                for w in ws:
                    a = (np.int64(kmin) + np.int64(64 * int(w)) + np.arange(64, dtype=np.int64)).view(np.uint64)
                    b = (np.int64(kmin) + np.int64(64 * (int(w) % period)) + np.arange(64, dtype=np.int64)).view(np.uint64)
                    assert np.array_equal(po.partition_of(a, n), po.partition_of(b, n))


def test_oracle_local_plans_match_reference_scan(tmp_path):
    """plan_oracle.execute_local (the Q6-analog restatement) against the reference's own
    read_blocking + predicate + sums (tests/golden/local.json), per node."""
    import json as _json
    local = _json.load(open(os.path.join(os.path.dirname(__file__), "golden", "local.json")))
    n = 0
    for r in local["results"]:
        if r["scale"] > 0.1:
            continue
        d = str(tmp_path / r["case"])
        oracle.gen_tpch(d, r["scale"], r["nodes"], r["nodes"], r["seed"], r["codec"])
        got = po.execute_local(_json.dumps(local["plans"][r["plan"]]), d, r["nodes"])
        for k, want in enumerate(r["per_node"]):
            s = po.summary([got[k]])
            assert s["rows"] == want["rows"], (r["case"], k)
            if want["rows"]:
                assert s["colsums"] == want["colsums"] and s["rowhash"] == want["rowhash"], (r["case"], k)
        n += 1
    assert n >= 6


def test_oracle_synthetic_join_plans_match_reference(tmp_path):
    """The oracle's executor restatement on the synthetic-join tables (all plan shapes: grouped
    with build-side sums, global, no aggregate, build+probe predicates) against the reference's
    own results (tests/golden/synthetic.json)."""
    import json as _json
    import paper_2512_02862_b200 as psg  # the generator only (byte-identical, test_abi.py)
    syn = _json.load(open(os.path.join(os.path.dirname(__file__), "golden", "synthetic.json")))
    seen = set()
    for r in syn["results"]:
        if r["case"] in seen:
            continue
        seen.add(r["case"])
        d = str(tmp_path / r["case"])
        psg.gen_workload("synthetic", d, devices=r["devices"], nodes=r["nodes"], seed=r["seed"], codec=r["codec"])
        got = po.summary(po.execute(_json.dumps(syn["plans"][r["plan"]]), d, r["nodes"]))
        assert (got["rows"], got["rowhash"], got["colsums"], got["per_node_rows"]) == \
            (r["rows"], r["rowhash"], r["colsums"], r["per_node_rows"]), r["case"]
