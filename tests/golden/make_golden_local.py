"""Golden fixtures for local plans (the Q6 analog; psg_execute_local) from the REFERENCE ITSELF.

The reference's execute_plan cannot run a plan without a shuffled join (pipeline.cpp:334-335), so
the Q6 analog is pinned through the reference's own scan operator: oracle/_ref/ref_driver scanagg
= read_blocking with the plan's predicate (scan.cpp:273-336, set up like the pybind `scan`,
bindings.cpp:139-155) per node shard, then the global-aggregate sums (HashAggregator::add
semantics). Development container only; writes tests/golden/local.json.
"""
import json
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
DRIVER = os.path.join(HERE, "..", "..", "oracle", "_ref", "ref_driver")

Q6_PRED = [{"col": "l_shipdate", "op": ">=", "value": 19940101}, {"col": "l_shipdate", "op": "<", "value": 19950101},
           {"col": "l_discount", "op": ">=", "value": 5}, {"col": "l_discount", "op": "<=", "value": 7}]


def local_plan(pred, sums):
    return {"buffer_target_bytes": 8388608, "io_workers": 4,
            "scans": [{"table": "lineitem", "paths": ["{data}/dev*/lineitem.node{node}.psto"], "predicate": pred}],
            "joins": [], "aggregate": {"group_by": "", "sums": sums}}


PLANS = {
    "q6": local_plan(Q6_PRED, ["l_extendedprice", "l_discount"]),
    "q6_dates": local_plan(Q6_PRED[:2], ["l_extendedprice"]),
    "q6_empty": local_plan([{"col": "l_shipdate", "op": ">", "value": 99999999}], ["l_extendedprice"]),
    "q6_count": local_plan([{"col": "l_discount", "op": "==", "value": 3}], []),
}
# (case, plan, scale, nodes, seed, codec)
CASES = [
    ("q6_s001_n1", "q6", 0.01, 1, 42, "identity"),
    ("q6_s01_n1", "q6", 0.1, 1, 42, "identity"),
    ("q6_s1_n1", "q6", 1.0, 1, 42, "identity"),
    ("q6_s01_n2", "q6", 0.1, 2, 42, "identity"),
    ("q6_s01_n1_block", "q6", 0.1, 1, 42, "block"),
    ("q6dates_s01_n1", "q6_dates", 0.1, 1, 42, "identity"),
    ("q6empty_s001_n1", "q6_empty", 0.01, 1, 42, "identity"),
    ("q6count_s001_n2", "q6_count", 0.01, 2, 7, "identity"),
]


def pred_arg(pred):
    return ";".join("%s:%s:%s" % (a["col"], a["op"], a["value"]) for a in pred)


def main():
    if not os.path.exists(DRIVER):
        sys.exit("build oracle/_ref first: oracle/build_ref.sh")
    tmp = tempfile.mkdtemp(prefix="golden_local_")
    results = []
    try:
        for name, pname, scale, nodes, seed, codec in CASES:
            d = os.path.join(tmp, "d")
            shutil.rmtree(d, ignore_errors=True)
            subprocess.run([DRIVER, "gen", "--out", d, "--scale", str(scale), "--nodes", str(nodes), "--devices",
                            str(nodes), "--seed", str(seed), "--codec", codec], check=True, capture_output=True)
            plan = PLANS[pname]
            per_node = []
            for k in range(nodes):
                path = os.path.join(d, "dev%d" % ((k + 1) % nodes), "lineitem.node%d.psto" % k)
                out = subprocess.run([DRIVER, "scanagg", "--paths", path, "--pred", pred_arg(plan["scans"][0]["predicate"]),
                                      "--sums", ",".join(plan["aggregate"]["sums"])],
                                     check=True, capture_output=True, text=True).stdout.strip().splitlines()[-1]
                r = json.loads(out)
                r.pop("seconds")
                per_node.append(r)
            results.append({"case": name, "plan": pname, "scale": scale, "nodes": nodes, "seed": seed, "codec": codec,
                            "per_node": per_node})
            print(name, [(r["rows"], r["colsums"]) for r in per_node], flush=True)
        json.dump({"plans": PLANS, "results": results}, open(os.path.join(HERE, "local.json"), "w"), indent=1)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    main()
