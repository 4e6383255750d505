"""Randomised plans vs the oracle on the GPU: predicates (all six operators, int and float
literals, several atoms per scan), projections, build- and probe-side sums, grouped / global /
no aggregate, all four modes. Seeded, so failures reproduce."""
import json
import random

import pytest

import paper_2512_02862_b200 as psg
from oracle import plan_oracle as po

pytestmark = pytest.mark.gpu

OPS = ["<", "<=", "==", "!=", ">=", ">"]
RANGES = {"c_mktsegment": (0, 4), "o_custkey": (0, 1500), "o_orderdate": (19920101, 19981228),
          "o_shippriority": (0, 4), "o_orderkey": (0, 15000), "l_orderkey": (0, 15000),
          "l_extendedprice": (90000, 189999), "l_discount": (0, 10), "l_shipdate": (19920101, 19981228)}


def _atoms(rng, cols):
    out = []
    for _ in range(rng.randint(0, 3)):
        c = rng.choice(cols)
        lo, hi = RANGES[c]
        v = rng.randint(lo, hi)
        if rng.random() < 0.2:
            v = v + 0.5
        out.append({"col": c, "op": rng.choice(OPS), "value": v})
    return out


def random_plan(rng):
    ocols = ["o_orderkey", "o_custkey", "o_orderdate", "o_shippriority"]
    lcols = ["l_orderkey", "l_extendedprice", "l_discount", "l_shipdate"]
    opred = _atoms(rng, ["o_orderdate", "o_shippriority", "o_custkey"])
    lpred = _atoms(rng, ["l_shipdate", "l_discount", "l_extendedprice"])
    cpred = _atoms(rng, ["c_mktsegment"])
    scans = [{"table": "customer", "paths": ["{data}/dev*/customer.psto"], "replicated": True, "predicate": cpred},
             {"table": "orders", "paths": ["{data}/dev*/orders.node{node}.psto"], "predicate": opred},
             {"table": "lineitem", "paths": ["{data}/dev*/lineitem.node{node}.psto"], "predicate": lpred}]
    if rng.random() < 0.5:  # projection must keep keys and predicate columns
        need = {"o_orderkey", "o_custkey"} | {a["col"] for a in opred}
        scans[1]["columns"] = [c for c in ocols if c in need or rng.random() < 0.5]
    if rng.random() < 0.5:
        need = {"l_orderkey"} | {a["col"] for a in lpred}
        scans[2]["columns"] = [c for c in lcols if c in need or rng.random() < 0.6]
    joins = [{"id": "co", "build": "customer", "probe": "orders", "build_key": "c_custkey", "probe_key": "o_custkey",
              "mode": "replicated"},
             {"id": "res", "build": "co", "probe": "lineitem", "build_key": "o_orderkey", "probe_key": "l_orderkey",
              "mode": "shuffle"}]
    cand_extra = ["c_mktsegment"]
    shape = rng.random()
    if shape < 0.15:  # no local join: orders shuffled directly
        joins = [dict(joins[1], build="orders")]
        cand_extra = []
    elif shape < 0.3:  # a chain of two local joins on the build side (customer read twice)
        scans.append({"table": "cust2", "paths": ["{data}/dev*/customer.psto"], "replicated": True,
                      "predicate": _atoms(rng, ["c_mktsegment"])})
        joins = [joins[0], {"id": "co2", "build": "cust2", "probe": "co", "build_key": "c_custkey",
                            "probe_key": "o_custkey", "mode": "replicated"}, dict(joins[1], build="co2")]
        cand_extra = ["c_mktsegment"]
    elif shape < 0.45:  # a local join on the probe side (lineitem rows whose order key is a customer key)
        scans.append({"table": "cust3", "paths": ["{data}/dev*/customer.psto"], "replicated": True,
                      "predicate": _atoms(rng, ["c_mktsegment"])})
        joins = [joins[0], {"id": "lc", "build": "cust3", "probe": "lineitem", "build_key": "c_custkey",
                            "probe_key": "l_orderkey", "mode": "replicated"}, dict(joins[1], probe="lc")]
    plan = {"scans": scans, "joins": joins}
    r = rng.random()
    if r < 0.8:
        ocols_p = scans[1].get("columns", ocols)
        lcols_p = scans[2].get("columns", lcols)
        cand = cand_extra + [c for c in ocols_p if c != "o_orderkey"] + list(lcols_p)
        sums = rng.sample(cand, rng.randint(0, min(4, len(cand))))
        plan["aggregate"] = {"group_by": "l_orderkey" if r < 0.65 else "", "sums": sums}
    return plan


@pytest.fixture(scope="module")
def data(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("fz") / "d")
    psg.gen_workload("tpch", d, devices=1, nodes=1, scale=0.01, seed=3, row_group_bytes=64 << 10, codec="identity")
    return d


@pytest.fixture(scope="module")
def ctx():
    c = psg.Context(0)
    c.set_ingest(io_threads=3, batch_bytes=256 << 10)
    yield c
    c.close()


@pytest.mark.parametrize("seed", range(60))
def test_random_plan_matches_oracle(ctx, data, seed):
    rng = random.Random(seed)
    plan = random_plan(rng)
    mode = rng.choice(list(psg.MODES))
    want = po.summary(po.execute(json.dumps(plan), data, 1))
    got = ctx.execute_plan(plan, data, mode)
    s = po.summary([(got.schema, got.rows)])
    assert s == want, (seed, mode, json.dumps(plan))


def random_dup_plan(rng):
    """Replicated build sides with repeated keys (HashTable::build keeps duplicates and the probe
    emits every match, ops.cpp:105-222): orders replicated and built on o_custkey."""
    def atoms(cols):  # at most one range atom per scan, so most plans return rows
        if rng.random() < 0.4:
            return []
        c = rng.choice(cols)
        lo, hi = RANGES[c]
        return [{"col": c, "op": rng.choice(["<", "<=", ">=", ">", "!="]), "value": rng.randint(lo, hi)}]

    opred = atoms(["o_orderdate", "o_shippriority"])
    lpred = atoms(["l_shipdate", "l_discount", "l_extendedprice"])
    cpred = atoms(["c_mktsegment"])
    scans = [{"table": "orders", "paths": ["{data}/dev*/orders.node{node}.psto"], "replicated": True, "predicate": opred},
             {"table": "customer", "paths": ["{data}/dev*/customer.psto"], "predicate": cpred},
             {"table": "lineitem", "paths": ["{data}/dev*/lineitem.node{node}.psto"], "predicate": lpred}]
    oc = {"id": "oc", "build": "orders", "probe": "customer", "build_key": "o_custkey", "probe_key": "c_custkey",
          "mode": "replicated"}
    if rng.random() < 0.5:  # expanding chain on the shuffle build side
        joins = [oc, {"id": "res", "build": "oc", "probe": "lineitem", "build_key": "o_orderkey",
                      "probe_key": "l_orderkey", "mode": "shuffle"}]
        group = "l_orderkey"
    else:  # ... on the shuffle probe side (lineitem shuffled as the build side, keys repeat)
        joins = [oc, {"id": "res", "build": "lineitem", "probe": "oc", "build_key": "l_orderkey",
                      "probe_key": "o_orderkey", "mode": "shuffle"}]
        group = "o_orderkey"
    if rng.random() < 0.3:  # a second, unique-key local join after the expanding one
        scans.append({"table": "cust2", "paths": ["{data}/dev*/customer.psto"], "replicated": True,
                      "predicate": atoms(["c_mktsegment"])})
        j2 = {"id": "oc2", "build": "cust2", "probe": "oc", "build_key": "c_custkey", "probe_key": "c_custkey",
              "mode": "replicated"}
        joins = [joins[0], j2] + [dict(joins[1], **({"build": "oc2"} if joins[1]["build"] == "oc" else {"probe": "oc2"}))]
    plan = {"scans": scans, "joins": joins}
    r = rng.random()
    if r < 0.85:
        cand = ["l_extendedprice", "l_discount", "l_shipdate", "o_orderdate", "o_shippriority", "c_mktsegment"]
        plan["aggregate"] = {"group_by": group if r < 0.7 else "", "sums": rng.sample(cand, rng.randint(0, 4))}
    return plan


@pytest.mark.parametrize("seed", range(24))
def test_random_duplicate_key_plan_matches_oracle(ctx, data, seed):
    rng = random.Random(1000 + seed)
    plan = random_dup_plan(rng)
    mode = rng.choice(list(psg.MODES))
    want = po.summary(po.execute(json.dumps(plan), data, 1))
    got = ctx.execute_plan(plan, data, mode)
    s = po.summary([(got.schema, got.rows)])
    assert s == want, (seed, mode, json.dumps(plan))
