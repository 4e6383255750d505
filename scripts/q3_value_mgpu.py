"""A/B driver at N GPUs (run under torchrun): stage each rank's SF100 shards in HBM once, time K
staged queries (device time, max over ranks), report the dominant kernel, shuffle bytes and
exchange time, and check the summed result checksum against tests/golden/sf100.json.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/q3_value_mgpu.py [--steps 10]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=float, default=100.0)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--tag", default="")
ap.add_argument("--data-dir", default="/tmp/psg_bench")
ap.add_argument("--clocks", action="store_true", help="run bench.py's nvidia-smi clock sampler during the timed loop")
a = ap.parse_args()
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
root = bench.data_root_for(a.data_dir, a.scale, "identity")
if rank == 0:
    bench.gen_data_subprocess(root, a.scale, bench.SHARDS)
dist.barrier()
import paper_2512_02862_b200 as psg  # noqa: E402

obj = [psg.Context.unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
ctx = psg.Context(local, rank, world, obj[0])
ctx.set_ingest(io_threads=8, batch_bytes=64 << 20)
shards = [k for k in range(bench.SHARDS) if k % world == rank]
st = ctx.stage_plan(bench.plan_for(shards, 8), root)
for _ in range(a.warmup):
    st.run(want_rows=False)
q, k, x, rb = [], [], [], []
clk = bench.Clocks(",".join(str(i) for i in range(world)) if local == 0 else None)
if a.clocks:
    clk.__enter__()
for _ in range(a.steps):
    dist.barrier()
    s = st.run(want_rows=False)
    q.append(s["device_ms"])
    k.append(s["probe_kernel_ms"] / max(1, s["probe_kernel_launches"]))
    x.append(s["exchange_ms"])
    rb.append(s["bytes_received"])
if a.clocks:
    clk.__exit__()
dist.barrier()
res = st.run(want_rows=True)
cs = res.checksum()
t = torch.tensor([statistics.median(q), statistics.median(k), statistics.median(x), statistics.mean(q), max(q)], device="cuda",
                 dtype=torch.float64)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
h = torch.tensor([int(cs["rowhash"], 16) - (1 << 64) if int(cs["rowhash"], 16) >= (1 << 63) else int(cs["rowhash"], 16),
                  cs["rows"]], device="cuda", dtype=torch.int64)
dist.all_reduce(h)
g = bench.golden(a.scale)
rowhash = "%016x" % (int(h[0].item()) % (1 << 64))
if rank == 0:
    print(json.dumps({"tag": a.tag, "n": world, "query_ms": round(t[0].item(), 4), "query_ms_mean": round(t[3].item(), 4), "query_ms_max": round(t[4].item(), 4), "probe_ms": round(t[1].item(), 4),
                      "exchange_ms": round(t[2].item(), 4), "recv_bytes_rank0": int(statistics.median(rb)),
                      "agg_table": s["agg_table"], "launches": s["kernel_launches"],
                      "parity": g is not None and rowhash == g["rowhash"] and int(h[1].item()) == g["groups"]}), flush=True)
ctx.close()
dist.destroy_process_group()
