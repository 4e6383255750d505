"""Plan parsing/validation parity (CPU): psg_plan_resolve against the reference's own
QueryPlan::from_json_text + validate (pipeline.cpp:108-196), pinned by tests/golden/plans.json
(made by tests/golden/make_golden_plans.py from oracle/_ref). The reference raises nlohmann
json exceptions for malformed/mistyped JSON; the C ABI reports those as InvalidInput."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import paper_2512_02862_b200 as psg  # noqa: E402
from make_golden_plans import make_tree  # noqa: E402

GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "plans.json")))


@pytest.fixture(scope="module")
def tree(tmp_path_factory):
    root = str(tmp_path_factory.mktemp("plantree"))
    make_tree(root)
    return root


@pytest.mark.parametrize("name", sorted(GOLD["cases"]))
def test_plan_resolution_matches_reference(tree, name):
    case = GOLD["cases"][name]
    want = case["reference"]
    try:
        got = psg.resolve_plan(case["plan"], tree, case["node"], case["nodes"])
        got = json.loads(json.dumps(got).replace(tree, "{root}"))
    except psg.PsgError as e:
        got = {"error": e.kind}
    if want.get("error") == "json":
        assert got == {"error": "InvalidInput"}
    else:
        assert got == want


def test_glob_with_several_stars_in_one_component(tree):
    plan = {"scans": [{"table": "t", "paths": ["{data}/dev*/*node*.psto"]}]}
    got = psg.resolve_plan(plan, tree)["scans"][0]["paths"]
    want = sorted(os.path.join(tree, p) for p in GOLD["tree"] if p.startswith("dev") and "node" in p)
    assert got == want
