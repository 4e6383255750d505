"""Golden plan resolutions from the REFERENCE ITSELF (QueryPlan::from_json_text + validate,
/root/reference/proj/src/pipeline.cpp:108-196) via `oracle/_ref/ref_driver plan`.

Builds a fixed directory tree (TREE below) under a temp root, resolves every case in CASES with the
reference, and stores the result (resolved scans with the root replaced by "{root}", or the
reference's exception class) in plans.json. tests/test_plan.py rebuilds the tree and checks
psg_plan_resolve against it. Development container only (needs oracle/_ref)."""
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
DRIVER = os.path.join(HERE, "..", "..", "oracle", "_ref", "ref_driver")

TREE = ["dev0/customer.psto", "dev0/orders.node0.psto", "dev1/orders.node1.psto", "dev1/lineitem.node0.psto",
        "dev0/lineitem.node1.psto", "dev2/orders.node2.psto", "dev10/orders.node0.psto", "devx/readme.txt",
        "a/b1/c.psto", "a/b2/c.psto", "a/b2/d.psto", "a/xb3/c.psto", "a/b4/", "flat_0.psto", "flat_1.psto"]


def scan(table, paths, replicated=False, **kw):
    d = {"table": table, "paths": paths}
    if replicated:
        d["replicated"] = True
    d.update(kw)
    return d


def q3(o_paths, l_paths):
    return {"scans": [scan("customer", ["{data}/dev*/customer.psto"], True),
                      scan("orders", o_paths), scan("lineitem", l_paths)],
            "joins": [{"id": "co", "build": "customer", "probe": "orders", "build_key": "c_custkey",
                       "probe_key": "o_custkey", "mode": "replicated"},
                      {"id": "res", "build": "co", "probe": "lineitem", "build_key": "o_orderkey",
                       "probe_key": "l_orderkey", "mode": "shuffle"}],
            "aggregate": {"group_by": "l_orderkey", "sums": ["l_extendedprice"]}}


def cases():
    c = {}
    c["q3_node0"] = (q3(["{data}/dev*/orders.node{node}.psto"], ["{data}/dev*/lineitem.node{node}.psto"]), 0, 2)
    c["q3_node1"] = (q3(["{data}/dev*/orders.node{node}.psto"], ["{data}/dev*/lineitem.node{node}.psto"]), 1, 2)
    c["nodes_placeholder"] = (q3(["{data}/dev*/orders.node{node}.psto"], ["{data}/dev{nodes}/lineitem.node0.psto"]), 0, 1)
    c["literal_paths"] = (q3(["{data}/dev0/orders.node0.psto", "{data}/dev1/orders.node1.psto"],
                             ["{data}/dev1/lineitem.node0.psto"]), 0, 1)
    c["nested_wildcards"] = ({"scans": [scan("t", ["{data}/a/*/c.psto"])]}, 0, 1)
    c["prefix_suffix"] = ({"scans": [scan("t", ["{data}/a/b*/c.psto", "{data}/flat_*.psto"])]}, 0, 1)
    c["two_components"] = ({"scans": [scan("t", ["{data}/a/b*/*.psto"])]}, 0, 1)
    c["no_match"] = (q3(["{data}/dev*/orders.node7.psto"], ["{data}/dev*/lineitem.node0.psto"]), 0, 1)
    c["missing_literal"] = ({"scans": [scan("t", ["{data}/nope.psto"])]}, 0, 1)
    c["no_scans"] = ({"scans": []}, 0, 1)
    p = q3(["{data}/dev*/orders.node0.psto"], ["{data}/dev*/lineitem.node0.psto"])
    p["scans"][0].pop("replicated")
    c["local_join_not_replicated"] = (p, 0, 1)
    p = q3(["{data}/dev*/orders.node0.psto"], ["{data}/dev*/lineitem.node0.psto"])
    p["joins"][0]["mode"] = "shuffle"
    c["two_shuffles"] = (p, 0, 1)
    p = q3(["{data}/dev*/orders.node0.psto"], ["{data}/dev*/lineitem.node0.psto"])
    p["aggregate"]["group_by"] = "o_orderkey"
    c["group_by_not_probe_key"] = (p, 0, 1)
    p = q3(["{data}/dev*/orders.node0.psto"], ["{data}/dev*/lineitem.node0.psto"])
    p["aggregate"]["group_by"] = ""
    c["global_aggregate"] = (p, 0, 1)
    p = q3(["{data}/dev*/orders.node0.psto"], ["{data}/dev*/lineitem.node0.psto"])
    p["joins"][0]["build"] = "nation"
    c["unknown_build_scan"] = (p, 0, 1)
    p = q3(["{data}/dev*/orders.node0.psto"], ["{data}/dev*/lineitem.node0.psto"])
    del p["joins"][1]["probe_key"]
    c["missing_join_key"] = (p, 0, 1)
    c["bad_json"] = ("{\"scans\": [", 0, 1)
    p = q3(["{data}/dev*/orders.node0.psto"], ["{data}/dev*/lineitem.node0.psto"])
    p["scans"][1]["predicate"] = [{"col": "o_orderdate", "op": "~", "value": 1}]
    c["bad_operator"] = (p, 0, 1)
    p = q3(["{data}/dev*/orders.node0.psto"], ["{data}/dev*/lineitem.node0.psto"])
    p["budget_mb"] = 64
    p["io_workers"] = 3
    p["scans"][2]["columns"] = ["l_orderkey", "l_extendedprice"]
    c["options"] = (p, 0, 1)
    return c


def make_tree(root):
    for rel in TREE:
        path = os.path.join(root, rel)
        if rel.endswith("/"):
            os.makedirs(path, exist_ok=True)
            continue
        os.makedirs(os.path.dirname(path), exist_ok=True)
        open(path, "wb").close()


def main():
    out = {"tree": TREE, "cases": {}}
    with tempfile.TemporaryDirectory() as root:
        make_tree(root)
        for name, (plan, node, nodes) in cases().items():
            text = plan if isinstance(plan, str) else json.dumps(plan)
            r = subprocess.run([DRIVER, "plan", "--plan-json", text, "--data", root, "--node", str(node),
                                "--nodes", str(nodes)], capture_output=True, text=True, check=True)
            got = json.loads(r.stdout.replace(root, "{root}"))
            out["cases"][name] = {"plan": text, "node": node, "nodes": nodes, "reference": got}
            print(name, json.dumps(got)[:120])
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    sys.exit(main())
