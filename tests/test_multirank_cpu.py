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


# ---------------------------------------------------------------------------------------------
# The engine's shuffle protocol, driven from N gloo ranks on CPU. Each rank partitions its rows
# with the engine's partition_of, all-gathers its destination histogram (the count matrix the GPU
# ranks all-gather over NCCL), derives its send/receive layout with the engine's own
# psg_shuffle_plan, packs rows with psg_pack_plan's layout from all-reduced bounds, and exchanges
# the destination-major slab over gloo send/recv exactly as the engine's grouped ncclSend/ncclRecv
# does. The waves are voted with a MAX all-reduce (the kDoneFlag vote, pipeline.cpp:696-722) so a
# rank with fewer batches keeps joining with empty waves.
def _shuffle_worker(rank, world, port, out_dir):
    import sys
    import numpy as np
    import torch
    sys.path.insert(0, ROOT)
    import paper_2512_02862_b200 as psg
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(100 + rank)
    nbatches = 2 + rank  # ranks disagree on their batch counts
    waves = torch.tensor([nbatches])
    dist.all_reduce(waves, op=dist.ReduceOp.MAX)
    # all-reduced bounds of the shipped columns (key, price, discount) -> one packed word per row
    keys_all = [rng.integers(0, 150_000, 5000 + 700 * b) for b in range(nbatches)]
    price_all = [rng.integers(90_000, 190_000, len(k)) for k in keys_all]
    disc_all = [rng.integers(0, 11, len(k)) for k in keys_all]
    lo = torch.tensor([~int(min(k.min() for k in keys_all)), ~int(min(p.min() for p in price_all)),
                       ~int(min(d.min() for d in disc_all))], dtype=torch.int64)
    hi = torch.tensor([int(max(k.max() for k in keys_all)), int(max(p.max() for p in price_all)),
                       int(max(d.max() for d in disc_all))], dtype=torch.int64)
    dist.all_reduce(lo, op=dist.ReduceOp.MAX)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    L = psg.pack_plan(~lo.numpy(), hi.numpy())
    layouts = [None] * world
    dist.all_gather_object(layouts, (L["fits"], L["min"].tolist(), L["shift"].tolist(), L["mask"].tolist()))
    got_rows, sent_rows = [], 0
    for w in range(int(waves.item())):
        have = w < nbatches
        k = keys_all[w] if have else np.zeros(0, np.int64)
        cols = [k, price_all[w], disc_all[w]] if have else [k, k, k]
        dest = psg.partition_of(k, world).astype(np.int64)
        hist = torch.tensor(np.bincount(dest, minlength=world), dtype=torch.int64)
        gathered = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, hist)
        matrix = torch.stack(gathered).numpy().astype(np.uint64)
        so, ro, sr, rr = psg.shuffle_plan(matrix, rank)
        # destination-major slab, stable within a destination (order-preserving partition,
        # core_ops_test.cpp:104-121); rows packed into one word
        order = np.argsort(dest, kind="stable")
        word = np.zeros(len(k), np.uint64)
        for c in range(3):
            word |= (cols[c].astype(np.uint64) - np.uint64(L["min"][c])) << np.uint64(L["shift"][c])
        slab = word[order]
        assert sr == len(k)
        recv = np.zeros(rr, np.uint64)
        reqs = []
        for p in range(world):
            sc = int(matrix[rank, p]); rc = int(matrix[p, rank])
            if p == rank:
                recv[int(ro[p]):int(ro[p]) + rc] = slab[int(so[p]):int(so[p]) + sc]
                continue
            if sc:
                reqs.append(dist.isend(torch.from_numpy(slab[int(so[p]):int(so[p]) + sc].view(np.int64).copy()), p))
            if rc:
                buf = torch.zeros(rc, dtype=torch.int64)
                reqs.append((dist.irecv(buf, p), buf, int(ro[p])))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                recv[r[2]:r[2] + len(r[1])] = r[1].numpy().view(np.uint64)
            else:
                r.wait()
        sent_rows += len(k)
        # unpack
        unpacked = [np.uint64(L["min"][c]) + ((recv >> np.uint64(L["shift"][c])) & np.uint64(L["mask"][c]))
                    for c in range(3)]
        got_rows.append(np.stack(unpacked, axis=1).astype(np.int64))
    got = np.concatenate(got_rows) if got_rows else np.zeros((0, 3), np.int64)
    np.save(os.path.join(out_dir, "recv%d.npy" % rank), got)
    sent = np.concatenate([np.stack([keys_all[b], price_all[b], disc_all[b]], axis=1) for b in range(nbatches)])
    np.save(os.path.join(out_dir, "sent%d.npy" % rank), sent)
    with open(os.path.join(out_dir, "meta%d.json" % rank), "w") as f:
        json.dump({"waves": int(waves.item()), "layouts_equal": all(l == layouts[0] for l in layouts),
                   "fits": bool(L["fits"])}, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shuffle_protocol_over_gloo(tmp_path, world):
    import numpy as np
    import paper_2512_02862_b200 as psg
    mp.spawn(_shuffle_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    metas = [json.load(open(tmp_path / ("meta%d.json" % r))) for r in range(world)]
    assert all(m["waves"] == 2 + world - 1 for m in metas)  # MAX vote over ranks
    assert all(m["layouts_equal"] and m["fits"] for m in metas)
    sent = np.concatenate([np.load(tmp_path / ("sent%d.npy" % r)) for r in range(world)])
    recvs = [np.load(tmp_path / ("recv%d.npy" % r)) for r in range(world)]
    for r, got in enumerate(recvs):  # every row lands on its owner, decoded exactly
        assert np.all(psg.partition_of(got[:, 0], world) == r)
    allgot = np.concatenate(recvs)
    key = lambda a: a[np.lexsort(a.T[::-1])]
    assert np.array_equal(key(allgot), key(sent))  # nothing lost, nothing duplicated


def test_shuffle_plan_offsets_and_pack_edge_cases():
    import numpy as np
    import paper_2512_02862_b200 as psg
    m = np.array([[3, 0, 5], [1, 1, 1], [0, 7, 2]], np.uint64)
    so, ro, sr, rr = psg.shuffle_plan(m, 1)
    assert so.tolist() == [0, 1, 2] and sr == 3
    assert ro.tolist() == [0, 0, 1] and rr == 8  # receives 0 from 0, 1 from 1, 7 from 2
    with pytest.raises(psg.PsgError):
        psg.shuffle_plan(m, 3)
    # 28 + 17 + 4 bits (Q3: key, price, discount) fit; a 64-bit span alone does not fit with others
    L = psg.pack_plan([0, 90000, 0], [150_000_000, 189_999, 10])
    assert L["fits"] and L["shift"].tolist() == [0, 28, 45]
    assert not psg.pack_plan([0, 0], [2 ** 62, 2 ** 10])["fits"]
    assert not psg.pack_plan([5, 0], [5, 10])["fits"]  # the key must be a real field
    assert psg.pack_plan([0, 1], [10, 0])["fits"]  # an empty column packs as an empty field
    # partition_of matches the oracle's restatement
    from oracle import plan_oracle as po
    k = np.random.default_rng(0).integers(-2 ** 40, 2 ** 40, 1000)
    assert np.array_equal(psg.partition_of(k, 3).astype(np.int64), po.partition_of(k.view(np.uint64), 3))
