"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Runs in the development container only (needs /root/reference and oracle/_ref/ref_driver, built by
oracle/build_ref.sh). The outputs are committed so the GPU box (which has no /root/reference) and
the CPU test suite can check both the oracle and the product against the reference's own results.

  gen_hashes.json : sha256 of every PSTO file the reference generator (gen_workload,
                    /root/reference/proj/src/bench.cpp:85-114) writes for a set of specs.
  results.json    : reference execute_plan results (row count, rowhash, column sums, rows per node)
                    for a set of plans/scales/node counts/modes, via run_socket_pipeline (1 node,
                    real threads) or run_sim_pipeline (n nodes, deterministic).
  q3_s001_rows.bin: raw result rows of the canonical plan at SF0.01 (u64 nrows, u64 ncols, words).
"""
import hashlib
import json
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
DRIVER = os.path.join(HERE, "..", "..", "oracle", "_ref", "ref_driver")

SCANS = lambda od, ld, extra_o="", extra_l="": [
    {"table": "customer", "paths": ["{data}/dev*/customer.psto"], "replicated": True,
     "predicate": [{"col": "c_mktsegment", "op": "==", "value": 1}]},
    {"table": "orders", "paths": ["{data}/dev*/orders.node{node}.psto"],
     "predicate": [{"col": "o_orderdate", "op": "<", "value": od}]},
    {"table": "lineitem", "paths": ["{data}/dev*/lineitem.node{node}.psto"],
     "predicate": [{"col": "l_shipdate", "op": ">", "value": ld}]},
]
JOINS = [
    {"id": "cust_orders", "build": "customer", "probe": "orders",
     "build_key": "c_custkey", "probe_key": "o_custkey", "mode": "replicated"},
    {"id": "result", "build": "cust_orders", "probe": "lineitem",
     "build_key": "o_orderkey", "probe_key": "l_orderkey", "mode": "shuffle"},
]


def q3(od=19950315, ld=19950315, sums=("l_extendedprice", "l_discount"), group_by="l_orderkey",
       buffer=8388608, aggregate=True, scans=None):
    p = {"buffer_target_bytes": buffer, "io_workers": 4, "scans": scans or SCANS(od, ld), "joins": JOINS}
    if aggregate:
        p["aggregate"] = {"group_by": group_by, "sums": list(sums)}
    return p


def plans():
    canon = q3()
    proj = q3()
    proj["scans"][2]["columns"] = ["l_orderkey", "l_extendedprice", "l_shipdate"]
    proj["scans"][1]["columns"] = ["o_orderkey", "o_custkey", "o_orderdate"]
    proj["aggregate"] = {"group_by": "l_orderkey", "sums": ["l_extendedprice", "o_orderdate", "c_mktsegment"]}
    multi = q3()
    multi["scans"][2]["predicate"] = [
        {"col": "l_shipdate", "op": ">=", "value": 19940101}, {"col": "l_shipdate", "op": "<", "value": 19950101},
        {"col": "l_discount", "op": ">=", "value": 5}, {"col": "l_discount", "op": "<=", "value": 7}]
    multi["scans"][1]["predicate"].append({"col": "o_shippriority", "op": "!=", "value": 3})
    glob_agg = q3(group_by="")
    empty = q3(ld=99999999)
    noagg = q3(od=19930301, ld=19980601, aggregate=False)
    fl = q3()  # float literal on an int column (literal_as<int64_t> truncation)
    fl["scans"][1]["predicate"] = [{"col": "o_orderdate", "op": "<", "value": 19950315.7}]
    # replicated build sides with DUPLICATE keys (HashTable::build keeps them, probe emits every
    # match, ops.cpp:105-222): orders replicated and built on o_custkey, probed by customer
    dup_build = {"buffer_target_bytes": 8388608, "io_workers": 4, "scans": [
        {"table": "orders", "paths": ["{data}/dev*/orders.node{node}.psto"], "replicated": True,
         "predicate": [{"col": "o_orderdate", "op": "<", "value": 19950315}]},
        {"table": "customer", "paths": ["{data}/dev*/customer.psto"],
         "predicate": [{"col": "c_mktsegment", "op": "==", "value": 1}]},
        {"table": "lineitem", "paths": ["{data}/dev*/lineitem.node{node}.psto"],
         "predicate": [{"col": "l_shipdate", "op": ">", "value": 19950315}]}],
        "joins": [{"id": "oc", "build": "orders", "probe": "customer", "build_key": "o_custkey",
                   "probe_key": "c_custkey", "mode": "replicated"},
                  {"id": "result", "build": "oc", "probe": "lineitem", "build_key": "o_orderkey",
                   "probe_key": "l_orderkey", "mode": "shuffle"}],
        "aggregate": {"group_by": "l_orderkey", "sums": ["l_extendedprice", "l_discount", "o_shippriority"]}}
    # ... and on the shuffle PROBE side: customer expands through replicated orders, then probes a
    # shuffled lineitem build side (whose keys repeat too)
    dup_probe = {"buffer_target_bytes": 8388608, "io_workers": 4, "scans": [
        {"table": "orders", "paths": ["{data}/dev*/orders.node{node}.psto"], "replicated": True,
         "predicate": [{"col": "o_orderdate", "op": "<", "value": 19940601}]},
        {"table": "customer", "paths": ["{data}/dev*/customer.psto"],
         "predicate": [{"col": "c_mktsegment", "op": "<=", "value": 1}]},
        {"table": "lineitem", "paths": ["{data}/dev*/lineitem.node{node}.psto"],
         "predicate": [{"col": "l_discount", "op": ">=", "value": 8}]}],
        "joins": [{"id": "oc", "build": "orders", "probe": "customer", "build_key": "o_custkey",
                   "probe_key": "c_custkey", "mode": "replicated"},
                  {"id": "result", "build": "lineitem", "probe": "oc", "build_key": "l_orderkey",
                   "probe_key": "o_orderkey", "mode": "shuffle"}],
        "aggregate": {"group_by": "o_orderkey", "sums": ["l_extendedprice", "o_shippriority", "c_mktsegment"]}}
    dup_noagg = json.loads(json.dumps(dup_build))
    del dup_noagg["aggregate"]
    dup_noagg["scans"][2]["predicate"] = [{"col": "l_shipdate", "op": ">", "value": 19980601}]
    return {
        "dup_build_chain": dup_build,
        "dup_probe_chain": dup_probe,
        "dup_no_aggregate": dup_noagg,
        "canonical": canon,
        "pipeline_test": q3(19940000, 19940000, buffer=262144),
        "acceptance": q3(19960000, 19930000, buffer=262144),
        "smoke_py": q3(19960000, 19930000, sums=("l_extendedprice",), buffer=131072),
        "projection_buildsums": proj,
        "multi_atom": multi,
        "global_agg": glob_agg,
        "empty": empty,
        "no_aggregate": noagg,
        "float_literal": fl,
    }


# (case name, plan name, scale, nodes, devices, seed, codec, rg_bytes, backend, modes)
CASES = [
    ("canon_s001_n1", "canonical", 0.01, 1, 1, 42, "identity", 1 << 20, "socket", ["overlapped"]),
    ("canon_s01_n1", "canonical", 0.1, 1, 1, 42, "identity", 1 << 20, "socket", ["overlapped"]),
    ("canon_s1_n1", "canonical", 1.0, 1, 1, 42, "identity", 1 << 20, "socket", ["overlapped", "blocking"]),
    ("canon_s001_n2", "canonical", 0.01, 2, 2, 42, "identity", 1 << 20, "sim", ["overlapped"]),
    ("canon_s001_n4", "canonical", 0.01, 4, 4, 42, "identity", 1 << 20, "sim", ["overlapped"]),
    ("canon_s001_n8", "canonical", 0.01, 8, 8, 42, "identity", 1 << 20, "sim", ["overlapped"]),
    ("canon_s01_n2", "canonical", 0.1, 2, 2, 42, "identity", 1 << 20, "sim", ["overlapped"]),
    ("pipetest_s0004_n2", "pipeline_test", 0.004, 2, 2, 42, "identity", 64 << 10, "sim",
     ["blocking", "fastio", "combined", "overlapped"]),
    ("accept_s002_n2_block", "acceptance", 0.02, 2, 2, 42, "block", 256 << 10, "sim", ["overlapped", "blocking"]),
    ("accept_s1_n1", "acceptance", 1.0, 1, 1, 42, "identity", 1 << 20, "socket", ["overlapped"]),
    ("pipetest_s1_n1", "pipeline_test", 1.0, 1, 1, 42, "identity", 1 << 20, "socket", ["overlapped"]),
    ("smoke_s0002_n2_seed11", "smoke_py", 0.002, 2, 2, 11, "identity", 1 << 20, "sim", ["overlapped"]),
    ("proj_s001_n2", "projection_buildsums", 0.01, 2, 2, 42, "identity", 1 << 20, "sim", ["overlapped"]),
    ("multi_s01_n1", "multi_atom", 0.1, 1, 1, 42, "identity", 1 << 20, "socket", ["overlapped"]),
    ("global_s001_n2", "global_agg", 0.01, 2, 2, 42, "identity", 1 << 20, "sim", ["overlapped"]),
    ("global_s001_n1", "global_agg", 0.01, 1, 1, 42, "identity", 1 << 20, "socket", ["overlapped"]),
    ("empty_s0002_n2", "empty", 0.002, 2, 1, 42, "identity", 1 << 20, "sim", ["overlapped", "blocking"]),
    ("noagg_s0002_n2", "no_aggregate", 0.002, 2, 2, 42, "identity", 64 << 10, "sim", ["overlapped"]),
    ("floatlit_s001_n1", "float_literal", 0.01, 1, 1, 42, "identity", 1 << 20, "socket", ["overlapped"]),
    ("canon_s001_n3_dev2", "canonical", 0.01, 3, 2, 42, "identity", 256 << 10, "sim", ["overlapped"]),
    ("dupbuild_s001_n1", "dup_build_chain", 0.01, 1, 1, 42, "identity", 1 << 20, "socket", ["overlapped", "blocking"]),
    ("dupbuild_s01_n1", "dup_build_chain", 0.1, 1, 1, 42, "identity", 256 << 10, "socket", ["overlapped"]),
    ("dupbuild_s001_n2", "dup_build_chain", 0.01, 2, 2, 42, "identity", 1 << 20, "sim", ["overlapped"]),
    ("dupprobe_s001_n1", "dup_probe_chain", 0.01, 1, 1, 42, "identity", 1 << 20, "socket", ["overlapped"]),
    ("dupprobe_s001_n2", "dup_probe_chain", 0.01, 2, 2, 42, "identity", 1 << 20, "sim", ["overlapped"]),
    ("dupnoagg_s001_n1", "dup_no_aggregate", 0.01, 1, 1, 42, "identity", 1 << 20, "sim", ["overlapped"]),
]

GEN_SPECS = [
    (0.01, 1, 1, 42, "identity", 1 << 20),
    (0.01, 2, 2, 42, "identity", 1 << 20),
    (0.01, 4, 4, 42, "identity", 1 << 20),
    (0.01, 2, 2, 42, "block", 1 << 20),
    (0.004, 2, 2, 42, "identity", 64 << 10),
    (0.002, 2, 2, 11, "identity", 1 << 20),
    (0.01, 3, 2, 42, "identity", 256 << 10),
]


def gen(out, scale, nodes, devices, seed, codec, rg):
    subprocess.run([DRIVER, "gen", "--out", out, "--scale", str(scale), "--nodes", str(nodes), "--devices",
                    str(devices), "--seed", str(seed), "--codec", codec, "--rg-bytes", str(rg)],
                   check=True, capture_output=True)


def main():
    if not os.path.exists(DRIVER):
        sys.exit("build oracle/_ref first: oracle/build_ref.sh")
    only = sys.argv[1:]  # case-name prefixes: regenerate just those cases, keep the rest of results.json
    tmp = tempfile.mkdtemp(prefix="golden_")
    try:
        hashes = []
        for spec in (GEN_SPECS if not only else []):
            d = os.path.join(tmp, "g")
            shutil.rmtree(d, ignore_errors=True)
            gen(d, *spec)
            files = {}
            for root, _dirs, fs in os.walk(d):
                for f in fs:
                    if f.endswith(".psto"):
                        p = os.path.join(root, f)
                        files[os.path.relpath(p, d)] = hashlib.sha256(open(p, "rb").read()).hexdigest()
            hashes.append({"scale": spec[0], "nodes": spec[1], "devices": spec[2], "seed": spec[3],
                           "codec": spec[4], "rg_bytes": spec[5], "files": dict(sorted(files.items()))})
        if not only:
            json.dump(hashes, open(os.path.join(HERE, "gen_hashes.json"), "w"), indent=1)

        ps = plans()
        results = []
        if only:
            keep = json.load(open(os.path.join(HERE, "results.json")))["results"]
            results = [r for r in keep if not any(r["case"].startswith(o) for o in only)]
        for name, pname, scale, nodes, devices, seed, codec, rg, backend, modes in CASES:
            if only and not any(name.startswith(o) for o in only):
                continue
            d = os.path.join(tmp, "d")
            shutil.rmtree(d, ignore_errors=True)
            gen(d, scale, nodes, devices, seed, codec, rg)
            text = json.dumps(ps[pname])
            for mode in modes:
                cmd = [DRIVER, "run", "--plan-json", text, "--data", d, "--mode", mode, "--backend", backend,
                       "--nodes", str(nodes)]
                if name == "canon_s001_n1":
                    cmd += ["--dump", os.path.join(HERE, "q3_s001_rows.bin")]
                for attempt in range(3):  # the socket harness occasionally aborts on a busy loopback port
                    pr = subprocess.run(cmd, capture_output=True, text=True)
                    if pr.returncode == 0:
                        break
                if pr.returncode != 0:
                    print("FAILED", name, mode, pr.stderr[-1500:], flush=True)
                pr.check_returncode()
                out = pr.stdout.strip().splitlines()[-1]
                r = json.loads(out)
                r.pop("seconds")
                results.append({"case": name, "plan": pname, "scale": scale, "nodes": nodes, "devices": devices,
                                "seed": seed, "codec": codec, "rg_bytes": rg, "backend": backend, "mode": mode, **r})
                print(name, mode, r["rows"], r["rowhash"], flush=True)
        json.dump({"plans": ps, "results": results}, open(os.path.join(HERE, "results.json"), "w"), indent=1)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    main()
