"""Cold-cache end to end (measurement tool): drops the page cache (root on the GPU box), then runs
one psg_execute_plan of the bench workload from NVMe; prints cold and warm e2e seconds.

  python scripts/cold_e2e.py [--codec identity|block]
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_02862_b200 as psg  # noqa: E402


def drop_caches():
    subprocess.run(["sync"], check=False)
    with open("/proc/sys/vm/drop_caches", "w") as f:
        f.write("3\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--codec", default="identity")
    ap.add_argument("--io-threads", type=int, default=16)
    a = ap.parse_args()
    root = os.path.join("/tmp/psg_bench", "sf100_n8" + ("" if a.codec == "identity" else "_" + a.codec))
    root, _ = bench.ensure_data(root, 100.0, bench.SHARDS, codec=a.codec)
    ctx = psg.Context(0)
    ctx.set_ingest(io_threads=a.io_threads, batch_bytes=64 << 20)
    plan = bench.plan_for(list(range(bench.SHARDS)), a.io_threads)
    out = {"codec": a.codec, "io_threads": a.io_threads}
    try:
        drop_caches()
        out["dropped"] = True
    except OSError as e:
        out["dropped"] = False
        out["drop_error"] = str(e)
    t = time.time()
    r = ctx.execute_plan(plan, root)
    out["cold_s"] = round(time.time() - t, 3)
    out["cold_groups"] = int(r.rows.shape[0])
    out["h2d_gb"] = round(r.stats["h2d_bytes"] / 1e9, 2)
    for _ in range(2):
        t = time.time()
        r = ctx.execute_plan(plan, root)
        out["warm_s"] = round(time.time() - t, 3)
    df = subprocess.run(["df", "-h", "/tmp"], capture_output=True, text=True).stdout.strip().splitlines()[-1]
    out["tmp_fs"] = df
    print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
