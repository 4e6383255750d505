"""Golden fixtures for the synthetic-join workload (gen_workload kind=synthetic) from the REFERENCE
ITSELF (oracle/_ref/ref_driver gen --kind synthetic / run). Development container only; writes
tests/golden/synthetic.json: file hashes of the generator output and execute_plan results of
shuffle-join plans over the build/probe tables (1 node real threads, 2-3 nodes sim)."""
import hashlib
import json
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
DRIVER = os.path.join(HERE, "..", "..", "oracle", "_ref", "ref_driver")

SCANS = [{"table": "build", "paths": ["{data}/dev*/build.node{node}.psto"]},
         {"table": "probe", "paths": ["{data}/dev*/probe.node{node}.psto"]}]
JOIN = [{"id": "j", "build": "build", "probe": "probe", "build_key": "bk", "probe_key": "pk", "mode": "shuffle"}]


def plan(aggregate=None, build_pred=None, probe_pred=None, buffer=262144):
    scans = json.loads(json.dumps(SCANS))
    if build_pred:
        scans[0]["predicate"] = build_pred
    if probe_pred:
        scans[1]["predicate"] = probe_pred
    p = {"buffer_target_bytes": buffer, "io_workers": 4, "scans": scans, "joins": JOIN}
    if aggregate is not None:
        p["aggregate"] = aggregate
    return p


PLANS = {
    "syn_agg": plan({"group_by": "pk", "sums": ["bp0", "pp0", "pp1"]}),
    "syn_global": plan({"group_by": "", "sums": ["bp1", "pp2"]}),
    "syn_noagg": plan(None, probe_pred=[{"col": "pp0", "op": "<", "value": 100000000}]),
    "syn_filtered": plan({"group_by": "pk", "sums": ["pp0"]},
                         build_pred=[{"col": "bp2", "op": ">=", "value": 250000000}],
                         probe_pred=[{"col": "pp0", "op": "<", "value": 500000000}]),
}
# (case, plan, nodes, devices, seed, codec, backend, modes)
CASES = [
    ("syn_agg_n1", "syn_agg", 1, 1, 42, "identity", "socket", ["overlapped", "blocking"]),
    ("syn_agg_n2", "syn_agg", 2, 2, 42, "identity", "sim", ["overlapped"]),
    ("syn_global_n2", "syn_global", 2, 2, 42, "identity", "sim", ["overlapped"]),
    ("syn_noagg_n1", "syn_noagg", 1, 1, 7, "identity", "socket", ["overlapped"]),
    ("syn_noagg_n2", "syn_noagg", 2, 2, 7, "identity", "sim", ["overlapped"]),
    ("syn_filtered_n1_block", "syn_filtered", 1, 1, 11, "block", "socket", ["overlapped"]),
    ("syn_filtered_n3", "syn_filtered", 3, 2, 11, "identity", "sim", ["overlapped"]),
]
GEN_SPECS = [(2, 2, 42, "identity"), (3, 2, 11, "block")]


def gen(d, nodes, devices, seed, codec):
    subprocess.run([DRIVER, "gen", "--kind", "synthetic", "--out", d, "--nodes", str(nodes), "--devices", str(devices),
                    "--seed", str(seed), "--codec", codec], check=True, capture_output=True)


def main():
    if not os.path.exists(DRIVER):
        sys.exit("build oracle/_ref first: oracle/build_ref.sh")
    tmp = tempfile.mkdtemp(prefix="golden_syn_")
    try:
        hashes = []
        for nodes, devices, seed, codec in GEN_SPECS:
            d = os.path.join(tmp, "g")
            shutil.rmtree(d, ignore_errors=True)
            gen(d, nodes, devices, seed, codec)
            files = {}
            for root, _dirs, fs in os.walk(d):
                for f in fs:
                    if f.endswith(".psto"):
                        p = os.path.join(root, f)
                        files[os.path.relpath(p, d)] = hashlib.sha256(open(p, "rb").read()).hexdigest()
            hashes.append({"nodes": nodes, "devices": devices, "seed": seed, "codec": codec,
                           "files": dict(sorted(files.items()))})
        results = []
        for name, pname, nodes, devices, seed, codec, backend, modes in CASES:
            d = os.path.join(tmp, "d")
            shutil.rmtree(d, ignore_errors=True)
            gen(d, nodes, devices, seed, codec)
            for mode in modes:
                out = subprocess.run([DRIVER, "run", "--plan-json", json.dumps(PLANS[pname]), "--data", d, "--mode", mode,
                                      "--backend", backend, "--nodes", str(nodes)],
                                     check=True, capture_output=True, text=True).stdout.strip().splitlines()[-1]
                r = json.loads(out)
                r.pop("seconds")
                results.append({"case": name, "plan": pname, "nodes": nodes, "devices": devices, "seed": seed,
                                "codec": codec, "backend": backend, "mode": mode, **r})
                print(name, mode, r["rows"], r["rowhash"], r["per_node_rows"], flush=True)
        json.dump({"plans": PLANS, "gen": hashes, "results": results}, open(os.path.join(HERE, "synthetic.json"), "w"),
                  indent=1)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    main()
