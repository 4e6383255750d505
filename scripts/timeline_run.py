"""Records an execution timeline (PSG_TIMELINE) of the warm end-to-end SF100 query: run under
torchrun for N > 1. Writes <out>.rank<r>.json (Chrome trace) and prints the summary on rank 0.

  PSG_TIMELINE=gpurun_out/tl python scripts/timeline_run.py [--codec block]"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_02862_b200 as psg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--codec", default="identity")
    a = ap.parse_args()
    world, rank, local = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), \
        int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    root = os.path.join("/tmp/psg_bench", "sf100_n8" + ("" if a.codec == "identity" else "_" + a.codec))
    if rank == 0:
        bench.ensure_data(root, 100.0, bench.SHARDS, codec=a.codec)
    nid = None
    if dist:
        dist.barrier()
        obj = [psg.Context.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    io = max(2, min(12, (os.cpu_count() or 4) // world))
    ctx = psg.Context(local, rank, world, nid)
    ctx.set_ingest(io_threads=io, batch_bytes=128 << 20)  # bench.py default
    plan = bench.plan_for([k for k in range(bench.SHARDS) if k % world == rank], io)
    for _ in range(3):  # the last run's timeline stays on disk
        if dist:
            dist.barrier()
        r = ctx.execute_plan(plan, root)
    ctx.close()
    if rank == 0:
        out = os.environ["PSG_TIMELINE"] + ".rank0.json"
        print("groups on rank 0:", r.rows.shape[0])
        subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "timeline_summary.py"), out])
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
