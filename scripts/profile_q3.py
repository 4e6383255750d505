"""Profiling driver: stage the Q3-analog plan in HBM and run it W+K times (one rank, no e2e leg).

  python scripts/profile_q3.py --scale 100 --warmup 1 --steps 1
Used under `ncu` for the launch list and the top-kernel capture; never a bench number."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_02862_b200 as psg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=float, default=100.0)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--data-dir", default="/tmp/psg_bench")
ap.add_argument("--no-semijoin", action="store_true")
a = ap.parse_args()
root, _ = bench.ensure_data(os.path.join(a.data_dir, "sf%g_n%d" % (a.scale, bench.SHARDS)), a.scale, bench.SHARDS)
ctx = psg.Context(0)
ctx.set_ingest(io_threads=16, batch_bytes=64 << 20)
if a.no_semijoin:
    ctx.set_semijoin(False)
st = ctx.stage_plan(bench.plan_for(list(range(bench.SHARDS)), 16), root)
for _ in range(a.warmup + a.steps):
    s = st.run(want_rows=False)
print(json.dumps(s))
