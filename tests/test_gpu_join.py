"""The distributed-join microbenchmark on the GPU (psg_run_synthetic_join, csrc/join.cpp): every
variant's joined rows equal the reference's run_sim_join rows (tests/golden/join.json, rowhash +
column sums; the multiset is independent of the node count) - build payload ++ probe columns."""
import json
import os

import pytest

import paper_2512_02862_b200 as psg
from oracle import plan_oracle as po

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "join.json")))


@pytest.fixture(scope="module")
def ctx():
    c = psg.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("variant", ["blocking", "blocking-opt", "chunking", "deferred"])
@pytest.mark.parametrize("gi", range(len(GOLD["joins"])))
def test_join_rows_match_reference(ctx, variant, gi):
    g = GOLD["joins"][gi]
    wl = g["workload"]
    st, res = ctx.run_synthetic_join(variant, stream_count=2 if variant in ("chunking", "deferred") else 1,
                                     chunk_rows=g["chunk_rows"], build_rows=wl["build_rows"],
                                     probe_rows=wl["probe_rows"], payload_cols=wl["payload"],
                                     hit_ratio=wl["hit_ratio"], seed=wl["seed"])
    s = po.summary([(res.schema, res.rows)])
    assert (s["rows"], s["rowhash"], s["colsums"]) == (g["rows"], g["rowhash"], g["colsums"])
    assert st["result_rows"] == g["rows"]
    names = [n for n, _t in res.schema]
    assert names == ["bp%d" % i for i in range(wl["payload"])] + ["pk"] + ["pp%d" % i for i in range(wl["payload"])]
    if variant in ("chunking", "deferred"):
        assert st["left_waves"] == max(1, -(-wl["build_rows"] // g["chunk_rows"]))
