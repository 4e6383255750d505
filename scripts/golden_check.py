"""Runs the reference's golden cases (tests/golden/results.json, local.json, synthetic.json) on
cuda:0 with whatever engine configuration the environment selects (e.g. PSG_JIT=0: the nvcc-built
interpreter kernel instead of query-compiled kernels) and prints one line per case; exit 1 on a
mismatch. Used by tests/test_gpu_interp.py."""
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_02862_b200 as psg  # noqa: E402
from oracle import plan_oracle as po  # noqa: E402


def main():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "results.json")))
    loc = json.load(open(os.path.join(ROOT, "tests", "golden", "local.json")))
    syn = json.load(open(os.path.join(ROOT, "tests", "golden", "synthetic.json")))
    ctx = psg.Context(0)
    ctx.set_ingest(io_threads=4, batch_bytes=2 << 20)
    bad = 0
    kinds = {}  # psg_stats.agg_table kind -> cases (4 = rank-indexed table)
    ovf = [0]  # rows that went through the bucket overflow list
    fused = [0]  # cases whose shuffle ran through the peer-slab path (PSG_SLAB_FAKE at one GPU)
    with tempfile.TemporaryDirectory() as tmp:
        cache = {}

        def data(scale, seed, rg, codec="identity"):
            k = (scale, seed, rg, codec)
            if k not in cache:
                d = os.path.join(tmp, "d%d" % len(cache))
                psg.gen_workload("tpch", d, devices=1, nodes=1, scale=scale, seed=seed, row_group_bytes=rg, codec=codec)
                cache[k] = d
            return cache[k]

        seen = set()
        for r in g["results"]:
            if r["scale"] > 0.1 or r["case"] in seen:
                continue
            seen.add(r["case"])
            res = ctx.execute_plan(g["plans"][r["plan"]], data(r["scale"], r["seed"], r["rg_bytes"], r["codec"]),
                                   r["mode"])
            s = po.summary([(res.schema, res.rows)])
            kinds[res.stats["agg_table"]] = kinds.get(res.stats["agg_table"], 0) + 1
            ovf[0] += res.stats["bucket_overflow"]
            fused[0] += res.stats.get("shuffle_fused", 0)
            if r["plan"] == "global_agg" and r["nodes"] > 1:
                ok = s["colsums"] == r["colsums"]
            else:
                ok = (s["rows"], s["rowhash"], s["colsums"]) == (r["rows"], r["rowhash"], r["colsums"])
            bad += not ok
            print("%-26s %s" % (r["case"], "OK" if ok else "BAD"), flush=True)
        for r in loc["results"]:
            if r["scale"] > 0.1:
                continue
            res = ctx.execute_local(loc["plans"][r["plan"]], data(r["scale"], r["seed"], 1 << 20, r["codec"]))
            rows = sum(x["rows"] for x in r["per_node"])
            cols = None
            for x in r["per_node"]:
                if x["rows"]:
                    v = [int(c) for c in x["colsums"]]
                    cols = v if cols is None else [(p + q) % (1 << 64) for p, q in zip(cols, v)]
            ok = res.rows.shape[0] == (1 if rows else 0) and (not rows or [int(c) for c in res.rows[0]] == cols)
            bad += not ok
            print("%-26s %s" % (r["case"], "OK" if ok else "BAD"), flush=True)
        for r in syn["results"]:
            if r["nodes"] != 1:
                continue
            d = os.path.join(tmp, "syn%d_%s" % (r["seed"], r["codec"]))
            if not os.path.exists(d):
                psg.gen_workload("synthetic", d, devices=1, nodes=1, seed=r["seed"], codec=r["codec"])
            res = ctx.execute_plan(syn["plans"][r["plan"]], d, r["mode"])
            s = po.summary([(res.schema, res.rows)])
            ok = (s["rows"], s["rowhash"], s["colsums"]) == (r["rows"], r["rowhash"], r["colsums"])
            bad += not ok
            print("%-26s %s" % (r["case"], "OK" if ok else "BAD"), flush=True)
    ctx.close()
    print("AGG_TABLES", json.dumps({str(k): v for k, v in sorted(kinds.items())}))
    print("BUCKET_OVERFLOW", ovf[0])
    print("SLAB_FUSED", fused[0])
    print("BAD", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
