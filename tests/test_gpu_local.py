"""Local plans (no shuffled join; psg_execute_local, the Q6 analog) on the GPU.

Pinned against the reference's own scan operator (tests/golden/local.json, made by
make_golden_local.py through read_blocking + predicate + HashAggregator sums) and against the
oracle's restatement (plan_oracle.execute_local) for plan shapes the reference cannot run at all
(local joins against replicated scans, float sums). The reference's execute_plan rejects such
plans with InvalidInput (pipeline.cpp:334-335); psg_execute_plan must keep doing so.
"""
import json
import os

import numpy as np
import pytest

import paper_2512_02862_b200 as psg
from oracle import plan_oracle as po

pytestmark = pytest.mark.gpu
LOCAL = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "local.json")))


@pytest.fixture(scope="module")
def ctx():
    c = psg.Context(0)
    c.set_ingest(io_threads=4, batch_bytes=4 << 20)
    yield c
    c.close()


@pytest.fixture(scope="module")
def ldata(tmp_path_factory):
    base = tmp_path_factory.mktemp("ldata")
    cache = {}

    def get(scale, seed=42, codec="identity"):
        key = (scale, seed, codec)
        if key not in cache:
            d = str(base / ("d%d" % len(cache)))
            psg.gen_workload("tpch", d, devices=1, nodes=1, scale=scale, seed=seed, codec=codec)
            cache[key] = d
        return cache[key]

    return get


def _totals(per_node):
    """Sum of the reference's per-node partial rows (the multiset is independent of node count)."""
    rows = sum(r["rows"] for r in per_node)
    cols = None
    for r in per_node:
        if r["rows"]:
            v = [int(x) for x in r["colsums"]]
            cols = v if cols is None else [(a + b) % (1 << 64) for a, b in zip(cols, v)]
    return rows, cols


@pytest.mark.parametrize("mode", ["overlapped", "blocking"])
def test_local_golden(ctx, ldata, mode):
    for r in LOCAL["results"]:
        res = ctx.execute_local(LOCAL["plans"][r["plan"]], ldata(r["scale"], r["seed"], r["codec"]), mode)
        nrows, cols = _totals(r["per_node"])
        want_rows = 1 if nrows else 0
        assert res.rows.shape[0] == want_rows, r["case"]
        if want_rows:
            assert [int(x) for x in res.rows[0]] == cols, r["case"]
        assert res.schema[0] == ("rows", "int64")


def test_local_plan_with_replicated_join_vs_oracle(ctx, ldata):
    # orders (filtered) joined with replicated customer (seg == 1) -> global sums; the reference
    # cannot express this plan, so the oracle's restatement is the checker
    plan = {"scans": [
        {"table": "customer", "paths": ["{data}/dev*/customer.psto"], "replicated": True,
         "predicate": [{"col": "c_mktsegment", "op": "==", "value": 1}]},
        {"table": "orders", "paths": ["{data}/dev*/orders.node{node}.psto"],
         "predicate": [{"col": "o_orderdate", "op": "<", "value": 19950315}]}],
        "joins": [{"id": "co", "build": "customer", "probe": "orders", "build_key": "c_custkey",
                   "probe_key": "o_custkey", "mode": "replicated"}],
        "aggregate": {"group_by": "", "sums": ["o_shippriority", "o_orderdate", "c_mktsegment"]}}
    d = ldata(0.1)
    res = ctx.execute_local(plan, d)
    want = po.execute_local(json.dumps(plan), d, 1)
    assert [n for n, _t in res.schema] == [n for n, _t in want[0][0]]
    assert np.array_equal(res.rows, want[0][1])


def test_local_float_sums_within_1e9(ctx, tmp_path):
    rng = np.random.default_rng(5)
    n = 300_000
    k = rng.integers(0, 1000, n)
    x = rng.normal(size=n) * 1e3
    path = str(tmp_path / "t.psto")
    psg.write_table(path, {"k": k.astype(np.int64), "x": x}, row_group_rows=4096)
    plan = {"scans": [{"table": "t", "paths": [path], "predicate": [{"col": "k", "op": "<", "value": 500},
                                                                    {"col": "x", "op": ">", "value": -250.5}]}],
            "joins": [], "aggregate": {"group_by": "", "sums": ["x", "k"]}}
    res = ctx.execute_local(plan, str(tmp_path))
    m = (k < 500) & (x > -250.5)
    assert res.rows[0][0] == m.sum()
    got = res.rows[0][1:2].view(np.float64)[0]
    assert abs(got - x[m].sum()) <= 1e-9 * np.abs(x[m]).sum()
    assert int(res.rows[0][2]) == int(k[m].sum())


def test_local_errors_match_reference(ctx, ldata, golden):
    d = ldata(0.01)
    q6 = LOCAL["plans"]["q6"]
    with pytest.raises(psg.PsgError) as e:  # the reference's execute_plan rejects no-shuffle plans
        ctx.execute_plan(q6, d)
    assert e.value.kind == "InvalidInput" and "shuffled join" in str(e.value)
    with pytest.raises(psg.PsgError) as e:  # and local execution rejects shuffle plans
        ctx.execute_local(golden["plans"]["canonical"], d)
    assert e.value.kind == "InvalidInput"
    grouped = json.loads(json.dumps(q6))
    grouped["aggregate"]["group_by"] = "l_orderkey"
    with pytest.raises(psg.PsgError):
        ctx.execute_local(grouped, d)
    bad = json.loads(json.dumps(q6))
    bad["aggregate"]["sums"] = ["no_such_column"]
    with pytest.raises(psg.PsgError) as e:
        ctx.execute_local(bad, d)
    assert e.value.kind == "UnknownColumn"
