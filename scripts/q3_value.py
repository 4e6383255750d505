"""A/B driver: stage the SF100 Q3-analog plan in HBM once and print the device time of K staged
queries and of their dominant probe kernel (CUDA events), plus the result checksum against
tests/golden/sf100.json. Engine knobs come from the environment (one process per variant).

  python scripts/q3_value.py [--steps 10 --warmup 3 --tag NAME]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=float, default=100.0)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--tag", default="")
ap.add_argument("--data-dir", default="/tmp/psg_bench")
a = ap.parse_args()
root = bench.data_root_for(a.data_dir, a.scale, "identity")
bench.gen_data_subprocess(root, a.scale, bench.SHARDS)
import paper_2512_02862_b200 as psg  # noqa: E402

ctx = psg.Context(0)
ctx.set_ingest(io_threads=12, batch_bytes=128 << 20)
st = ctx.stage_plan(bench.plan_for(list(range(bench.SHARDS)), 12), root)
for _ in range(a.warmup):
    st.run(want_rows=False)
q, k = [], []
for _ in range(a.steps):
    s = st.run(want_rows=False)
    q.append(s["device_ms"])
    k.append(s["probe_kernel_ms"] / max(1, s["probe_kernel_launches"]))
res = st.run(want_rows=True)
cs = res.checksum()
g = bench.golden(a.scale)
ok = g is not None and cs["rowhash"] == g["rowhash"] and cs["rows"] == g["groups"]
print(json.dumps({"tag": a.tag, "query_ms": round(statistics.median(q), 4), "query_ms_min": round(min(q), 4),
                  "probe_ms": round(statistics.median(k), 4), "probe_frac": round(19.2e9 / (statistics.median(k) / 1e3) / 1e9 / 6536.7, 4),
                  "launches": s["kernel_launches"], "agg_table": s["agg_table"], "parity": ok}), flush=True)
