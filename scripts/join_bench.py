"""Distributed-join microbenchmark (the reference's run_join variants, §Evaluation, on
B200s): times blocking / blocking-opt / chunking / deferred over one synthetic workload at N GPUs
(torchrun for N > 1) and prints one JSON line per variant - device time (max over ranks), host
waits, shuffled bytes and their effective rate.

  python scripts/join_bench.py [--build-rows 120000000 --probe-rows 320000000]
  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/join_bench.py"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_02862_b200 as psg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--build-rows", type=int, default=120_000_000)
ap.add_argument("--probe-rows", type=int, default=320_000_000)
ap.add_argument("--payload", type=int, default=3)
ap.add_argument("--hit-ratio", type=float, default=0.5)
ap.add_argument("--chunk-rows", type=int, default=8 << 20)
ap.add_argument("--streams", type=int, default=2)
ap.add_argument("--repeat", type=int, default=3)
ap.add_argument("--variants", default="blocking,blocking-opt,chunking,deferred")
a = ap.parse_args()
world, rank, local = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))
dist = None
nccl_id = None
if world > 1:
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [psg.Context.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    nccl_id = obj[0]
ctx = psg.Context(local, rank, world, nccl_id)


def red(x, op="max"):
    if not dist:
        return x
    import torch
    t = torch.tensor([float(x)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return t.item()


kw = dict(build_rows=a.build_rows, probe_rows=a.probe_rows, payload_cols=a.payload, hit_ratio=a.hit_ratio,
          collect_rows=False)
ctx.run_synthetic_join("deferred", a.streams, a.chunk_rows, **kw)  # generation + warm-up
for v in a.variants.split(","):
    k = 1 if v.startswith("blocking") else a.streams
    ms, wall, rows, rb, syncs = [], [], 0, 0, 0
    for _ in range(a.repeat):
        if dist:
            dist.barrier()
        st, _ = ctx.run_synthetic_join(v, k, a.chunk_rows, **kw)
        ms.append(st["device_ms"])
        wall.append(st["runtime_s"])
        rows, rb, syncs = st["result_rows"], st["bytes_received"], st["host_syncs"]
    dev = red(statistics.median(ms))
    recv = red(rb)
    total_rows = red(rows, "sum")
    wall_s = red(statistics.median(wall))  # (every rank: a collective)
    in_bytes = (a.build_rows + a.probe_rows) * (1 + a.payload) * 8
    if rank == 0:
        print(json.dumps({"variant": v, "n_gpus": world, "streams": k, "chunk_rows": a.chunk_rows,
                          "device_ms": round(dev, 3), "wall_s": round(wall_s, 4),
                          "result_rows": int(total_rows), "host_syncs": syncs, "recv_bytes_per_gpu": int(recv),
                          "shuffle_gbs": round(recv / 1e9 / (dev / 1e3), 1) if recv else None,
                          "input_gbs": round(in_bytes / 1e9 / (dev / 1e3), 1),
                          "workload": {"build_rows": a.build_rows, "probe_rows": a.probe_rows, "payload": a.payload,
                                       "hit_ratio": a.hit_ratio}}), flush=True)
ctx.close()
if dist:
    dist.destroy_process_group()
