"""Measurement tool: GPU inflate throughput on block-coded TPC-H data (not product code).

  python scripts/inflate_probe.py [--scale 10] [--steps 3]

Generates a block-codec dataset (node 0 of 1), then times (a) psg_stage_plan (read compressed
chunks -> HBM, one inflate launch over every chunk) and (b) execute_plan end to end, and prints the
decoded bytes / GB/s. Run under ncu with --metrics gpu__time_duration.sum to get the kernel time."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_02862_b200 as psg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=10.0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--dir", default="/tmp/psg_inflate")
    ap.add_argument("--batch-mb", type=int, default=64)
    a = ap.parse_args()
    d = os.path.join(a.dir, "sf%g_block" % a.scale)
    if not os.path.exists(os.path.join(d, "DONE")):
        t = time.time()
        psg.gen_workload("tpch", d, devices=1, nodes=1, scale=a.scale, seed=42, codec="block",
                         threads=3)
        open(os.path.join(d, "DONE"), "w").write("ok")
        print("gen %.1f s" % (time.time() - t), flush=True)
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "results.json")))
    plan = golden["plans"]["canonical"]
    ctx = psg.Context(0)
    ctx.set_ingest(io_threads=12, batch_bytes=a.batch_mb << 20)
    for i in range(a.steps):
        t = time.time()
        st = ctx.stage_plan(plan, d)
        ts = time.time() - t
        r = st.run(want_rows=False)
        print("stage %.3f s  run device %.2f ms  groups %d" % (ts, r["device_ms"], r["result_rows"]), flush=True)
        st.free()
    for i in range(a.steps):
        t = time.time()
        res = ctx.execute_plan(plan, d)
        te = time.time() - t
        s = res.stats
        print("e2e %.3f s  h2d %.2f GB  scanned %.2f GB  io_wait %.3f s  device %.1f ms groups %d" % (
            te, s["h2d_bytes"] / 1e9, s["ingest_bytes"] / 1e9, s["io_wait_s"], s["device_ms"], res.rows.shape[0]),
            flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
