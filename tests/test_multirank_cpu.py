"""Host-side N>1 logic on CPU with gloo (world_size 2): shard assignment and per-node semantics.

* bench.plan_for / rank r of N scans node shards k = r (mod N): every shard is scanned exactly
  once across ranks (gathered over gloo);
* the per-node result semantics the GPU ranks must reproduce (groups land on node
  partition_of(key) = ((key * 0x9E3779B97F4A7C15) >> 13) % N) hold in the oracle for the
  reference's own 2-node golden case.
"""
import json
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import bench
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shards = [k for k in range(bench.SHARDS) if k % world == rank]
    plan = bench.plan_for(shards, 2)
    mine = plan["scans"][1]["paths"] + plan["scans"][2]["paths"]
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    if rank == 0:
        flat = [p for ps in allp for p in ps]
        with open(os.path.join(out_dir, "paths.json"), "w") as f:
            json.dump(flat, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_every_shard_scanned_exactly_once(tmp_path, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    flat = json.load(open(tmp_path / "paths.json"))
    assert len(flat) == len(set(flat)) == 16  # 8 orders + 8 lineitem shards


def test_oracle_groups_land_on_partition_of_key(golden, datasets):
    import numpy as np
    from oracle import plan_oracle as po
    r = next(x for x in golden["results"] if x["case"] == "canon_s001_n2")
    d = datasets(r["scale"], r["nodes"], r["devices"])
    per_node = po.execute(json.dumps(golden["plans"]["canonical"]), d, 2)
    assert [rows.shape[0] for _s, rows in per_node] == r["per_node_rows"]
    for node, (_s, rows) in enumerate(per_node):
        assert np.all(po.partition_of(rows[:, 0], 2) == node)
