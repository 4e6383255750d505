"""Q6-analog measurement (BASELINE config 1: scan-filter-aggregate on lineitem; psg_execute_local).

  python scripts/q6_bench.py [--steps 5]

* SF1 (the reference's CPU-runnable config): GPU end to end (PSTO files -> HBM -> sums -> host)
  next to the reference's own single-worker read_blocking + predicate + sums (oracle/_ref
  ref_driver scanagg), results checked equal.
* SF100 (the bench dataset, all 8 lineitem shards on one GPU): GPU end to end.
Prints one JSON line. Measurement tool, not product code.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_02862_b200 as psg  # noqa: E402

PRED = [{"col": "l_shipdate", "op": ">=", "value": 19940101}, {"col": "l_shipdate", "op": "<", "value": 19950101},
        {"col": "l_discount", "op": ">=", "value": 5}, {"col": "l_discount", "op": "<=", "value": 7}]


def plan(paths):
    return {"scans": [{"table": "lineitem", "paths": paths, "predicate": PRED}], "joins": [],
            "aggregate": {"group_by": "", "sums": ["l_extendedprice", "l_discount"]}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--data-dir", default=os.environ.get("PSG_BENCH_DATA", "/tmp/psg_bench"))
    a = ap.parse_args()
    out = {"metric": "Q6-analog query seconds (scan-filter-aggregate on lineitem)"}
    ctx = psg.Context(0)
    ctx.set_ingest(io_threads=min(12, os.cpu_count() or 4), batch_bytes=64 << 20)
    # ---- SF1
    d1 = os.path.join(a.data_dir, "sf1_n1")
    if not os.path.exists(os.path.join(d1, "DONE")):
        psg.gen_workload("tpch", d1, devices=1, nodes=1, scale=1.0, seed=42, codec="identity")
        open(os.path.join(d1, "DONE"), "w").write("ok")
    p1 = plan(["{data}/dev0/lineitem.node0.psto"])
    ctx.execute_local(p1, d1)
    ts = []
    for _ in range(a.steps):
        t = time.time()
        r = ctx.execute_local(p1, d1)
        ts.append(time.time() - t)
    gpu_row = [int(x) for x in r.rows[0]]
    out["sf1_gpu_e2e_s"] = round(statistics.median(ts), 5)
    out["sf1_gpu_device_ms"] = round(r.stats["device_ms"], 3)
    out["sf1_result"] = gpu_row
    drv = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    if os.path.exists(drv):
        pred = ";".join("%s:%s:%s" % (x["col"], x["op"], x["value"]) for x in PRED)
        res = subprocess.run([drv, "scanagg", "--paths", os.path.join(d1, "dev0", "lineitem.node0.psto"), "--pred", pred,
                              "--sums", "l_extendedprice,l_discount", "--repeat", "3"], capture_output=True, text=True,
                             check=True).stdout.strip().splitlines()
        rr = [json.loads(x) for x in res]
        out["sf1_reference_cpu_s"] = round(statistics.median(x["seconds"] for x in rr), 5)
        out["sf1_reference_cores"] = 1
        out["sf1_reference_kind"] = "reference read_blocking + predicate + sums (single worker)"
        out["sf1_equal"] = [int(x) for x in rr[0]["colsums"]] == gpu_row
    # ---- SF100 (bench data)
    d100 = os.path.join(a.data_dir, "sf100_n8")
    if os.path.exists(os.path.join(d100, "DONE")):
        p100 = plan(["{data}/dev%d/lineitem.node%d.psto" % ((k + 1) % 8, k) for k in range(8)])
        ctx.execute_local(p100, d100)
        ts = []
        for _ in range(a.steps):
            t = time.time()
            r = ctx.execute_local(p100, d100)
            ts.append(time.time() - t)
        out["sf100_gpu_e2e_s"] = round(statistics.median(ts), 4)
        out["sf100_gpu_device_ms"] = round(r.stats["device_ms"], 2)
        out["sf100_h2d_gb"] = round(r.stats["h2d_bytes"] / 1e9, 2)
        out["sf100_ingest_gbs"] = round(r.stats["h2d_bytes"] / 1e9 / statistics.median(ts), 1)
        out["sf100_result"] = [int(x) for x in r.rows[0]]
    ctx.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
