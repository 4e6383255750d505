"""Staged (HBM-resident) Q3 SF100 under torchrun, one rank per GPU; prints per-run stats (rank 0)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2512_02862_b200 as psg  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 100.0
root = os.path.join("/tmp/psg_bench", "sf%g_n%d" % (scale, bench.SHARDS))
if rank == 0:
    bench.ensure_data(root, scale, bench.SHARDS)
dist.barrier()
obj = [psg.Context.unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
ctx = psg.Context(local, rank, world, obj[0])
ctx.set_ingest(io_threads=8, batch_bytes=64 << 20)
if os.environ.get("PSG_FUSED", "1") == "0":
    ctx.set_fused_shuffle(False)
st = ctx.stage_plan(bench.plan_for([k for k in range(bench.SHARDS) if k % world == rank], 8), root)
for i in range(4):
    dist.barrier()
    s = st.run(want_rows=False)
    if rank == 0:
        print("run", i, json.dumps({k: round(v, 4) if isinstance(v, float) else v for k, v in s.items()}), flush=True)
st.free()
ctx.close()
dist.destroy_process_group()
