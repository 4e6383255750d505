"""One storage-resident (e2e) query with PSG_TRACE phase timings; prints stats."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_02862_b200 as psg  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 100.0
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 16
batch_mb = int(sys.argv[3]) if len(sys.argv) > 3 else 64
root, _ = bench.ensure_data(os.path.join("/tmp/psg_bench", "sf%g_n%d" % (scale, bench.SHARDS)), scale, bench.SHARDS)
ctx = psg.Context(0)
ctx.set_ingest(io_threads=threads, batch_bytes=batch_mb << 20)
plan = bench.plan_for(list(range(bench.SHARDS)), threads)
for i in range(3):
    t = time.time()
    r = ctx.execute_plan(plan, root)
    t1 = time.time()
    print("run", i, "wall %.3f s" % (t1 - t), json.dumps({k: round(v, 4) if isinstance(v, float) else v
                                                      for k, v in r.stats.items()}), flush=True)
