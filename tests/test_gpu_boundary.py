"""The reference-side binding on the GPU: oracle/_ref/gpu_pipeline_harness (built here against the
unmodified reference headers by oracle/build_harness.sh; it travels to the GPU box) returns the
reference's own pystachio::PipelineResult from psg_execute_plan, for all four ExecModes, equal to
the reference engine's result on the same files (tests/golden/results.json, and oracle/_ref/
ref_driver run live on the box)."""
import json
import os
import subprocess

import pytest

import paper_2512_02862_b200 as psg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HARNESS = os.path.join(ROOT, "oracle", "_ref", "gpu_pipeline_harness")
REF = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


@pytest.fixture(scope="module")
def data(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("bd") / "d")
    psg.gen_workload("tpch", d, devices=1, nodes=1, scale=0.01, seed=42, codec="identity")
    return d


@pytest.mark.parametrize("mode", ["overlapped", "blocking", "fastio", "combined"])
def test_harness_pipeline_result_matches_reference(tmp_path, data, golden, mode):
    if not os.path.exists(HARNESS):
        pytest.fail("oracle/_ref/gpu_pipeline_harness missing: build() must run oracle/build_harness.sh")
    plan = tmp_path / "plan.json"
    plan.write_text(json.dumps(golden["plans"]["canonical"]))
    r = subprocess.run([HARNESS, "run", str(plan), data, mode], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    got = json.loads(r.stdout.strip().splitlines()[-1])
    want = next(x for x in golden["results"] if x["case"] == "canon_s001_n1")
    assert (got["rows"], got["rowhash"]) == (want["rows"], want["rowhash"])
    assert got["schema"] == ["l_orderkey", "rows", "sum_l_extendedprice", "sum_l_discount"]
    if os.path.exists(REF):  # the reference engine itself, live, on the same files
        ref = subprocess.run([REF, "run", "--plan", str(plan), "--data", data, "--mode", mode, "--backend", "sim"],
                             capture_output=True, text=True, timeout=300)
        rr = json.loads(ref.stdout.strip().splitlines()[-1])
        assert (got["rows"], got["rowhash"]) == (rr["rows"], rr["rowhash"])


def test_harness_budget_error_is_the_reference_class(tmp_path, data, golden):
    p = dict(golden["plans"]["canonical"], memory_budget_bytes=4096)
    plan = tmp_path / "plan.json"
    plan.write_text(json.dumps(p))
    r = subprocess.run([HARNESS, "run", str(plan), data, "overlapped"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 3, r.stdout + r.stderr
    assert "InfeasibleBudget" in r.stdout
    r = subprocess.run([HARNESS, "run", str(plan), data, "blocking"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 3 and ("MemoryExceeded" in r.stdout or "InfeasibleBudget" in r.stdout), r.stdout
