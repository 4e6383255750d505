"""Multi-GPU parity check (one rank per GPU, NCCL shuffle): run under torchrun.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/mgpu_check.py [--scale S]

Data is generated with nodes=N (the reference's layout), every rank executes the plan through
psg_execute_plan, and rank 0 checks each rank's rows against the reference's per-node results
(tests/golden/results.json where a case with nodes=N exists) and against the oracle otherwise.
Exit code 0 = all checks passed.
"""
import argparse
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2512_02862_b200 as psg  # noqa: E402
from oracle import plan_oracle as po  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=0.1)
    ap.add_argument("--modes", default="overlapped,blocking,staged")
    ap.add_argument("--fuzz", type=int, default=30, help="random plans (tests/test_gpu_fuzz.py) checked per node")
    ap.add_argument("--sf10", action="store_true", help="BASELINE config 2: canonical Q3 at SF10 vs the reference")
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "results.json")))
    base = tempfile.mkdtemp(prefix="mgpu_") if rank == 0 else None
    obj = [base]
    dist.broadcast_object_list(obj, src=0)
    base = obj[0]
    obj = [psg.Context.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = psg.Context(local, rank, world, obj[0])
    ctx.set_ingest(io_threads=4, batch_bytes=2 << 20)
    failures = []
    datasets = {}

    def run(plan, d, mode="overlapped"):
        """execute_plan in a streaming mode, or stage_plan + run ("staged": HBM-resident inputs,
        the chunked probe pipeline at N > 1)."""
        if mode == "staged":
            st = ctx.stage_plan(plan, d)
            try:
                return st.run()
            finally:
                st.free()
        return ctx.execute_plan(plan, d, mode)

    def data(scale, seed=42, rg=1 << 20, devices=None):
        key = (scale, seed, rg, devices)
        if key not in datasets:
            d = os.path.join(base, "d%d" % len(datasets))
            if rank == 0:
                psg.gen_workload("tpch", d, devices=devices or world, nodes=world, scale=scale, seed=seed,
                                 row_group_bytes=rg, codec="identity")
            dist.barrier()
            datasets[key] = d
        return datasets[key]

    cases = [("canonical", a.scale, 42, 1 << 20), ("acceptance", 0.02, 42, 256 << 10),
             ("projection_buildsums", 0.01, 42, 1 << 20), ("multi_atom", 0.1, 42, 1 << 20),
             ("global_agg", 0.01, 42, 1 << 20), ("empty", 0.002, 42, 1 << 20),
             ("no_aggregate", 0.002, 42, 64 << 10), ("smoke_py", 0.002, 11, 1 << 20),
             ("pipeline_test", 0.004, 42, 64 << 10)]
    variants = [(True, True), (True, False), (False, True), (False, False)]  # (fused NVLink, semi-join)
    for fused, semijoin in variants:
        ctx.set_semijoin(semijoin)
        try:
            ctx.set_fused_shuffle(fused)
        except psg.PsgError:
            if rank == 0:
                print("fused NVLink path unavailable; skipping fused variants")
            continue
        for pname, scale, seed, rg in cases:
            d = data(scale, seed, rg)
            plan = golden["plans"][pname]
            for mode in a.modes.split(","):
                try:
                    res = run(plan, d, mode)
                    mine = (res.schema, res.rows.copy())
                except psg.PsgError as e:
                    mine = ("error", str(e))
                allres = [None] * world
                dist.all_gather_object(allres, mine)
                if rank == 0:
                    if any(x[0] == "error" for x in allres):
                        failures.append((pname, mode, fused, semijoin, [x for x in allres if x[0] == "error"]))
                        continue
                    got = po.summary(allres)
                    g = [r for r in golden["results"] if r["plan"] == pname and r["nodes"] == world
                         and r["scale"] == scale and r["seed"] == seed and r["rg_bytes"] == rg]
                    if g:
                        want = {k: g[0][k] for k in ("rows", "rowhash", "colsums", "per_node_rows")}
                        src = "reference"
                    else:
                        want = po.summary(po.execute(json.dumps(plan), d, world))
                        src = "oracle"
                    ok = all(got[k] == want[k] for k in ("rows", "rowhash", "colsums", "per_node_rows"))
                    print("%-22s %-10s fused=%d semijoin=%d %-9s %s rows=%d per_node=%s" % (
                        pname, mode, fused, semijoin, src, "OK " if ok else "BAD", got["rows"], got["per_node_rows"]),
                        flush=True)
                    if not ok:
                        failures.append((pname, mode, fused, semijoin, got, want))
    # BASELINE config 2: Q3 at SF10 on N GPUs; the result multiset is independent of the node
    # count, so the union over ranks must equal the reference's SF10 golden
    if a.sf10:
        d = data(10.0, 42, 1 << 20)
        for mode in ("overlapped", "blocking", "staged"):
            res = run(golden["plans"]["canonical"], d, mode)
            allres = [None] * world
            dist.all_gather_object(allres, (res.schema, res.rows.copy()))
            if rank == 0:
                got = po.summary(allres)
                ok = (got["rows"], got["rowhash"]) == (1218662, "661bdb187378204d") and \
                    [int(x) for x in got["colsums"][1:]] == [2979547, 417235545352, 14897482]
                print("%-22s %-10s SF10      %s rows=%d per_node=%s" % ("canonical", mode, "OK " if ok else "BAD",
                                                                          got["rows"], got["per_node_rows"]), flush=True)
                if not ok:
                    failures.append(("sf10", mode, got))
    # randomised plans (all shapes of tests/test_gpu_fuzz.py) per node vs the oracle
    if a.fuzz:
        import importlib.util
        import random
        spec = importlib.util.spec_from_file_location("fz", os.path.join(ROOT, "tests", "test_gpu_fuzz.py"))
        fz = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(fz)
        d = data(0.01, 3, 64 << 10)
        nbad = 0
        for seed in range(a.fuzz):
            plan = fz.random_plan(random.Random(seed))
            try:
                res = run(plan, d, "staged" if seed % 2 else "overlapped")
                mine = (res.schema, res.rows.copy())
            except psg.PsgError as e:
                mine = ("error", str(e))
            allres = [None] * world
            dist.all_gather_object(allres, mine)
            if rank == 0:
                if any(x[0] == "error" for x in allres):
                    failures.append(("fuzz", seed, [x for x in allres if x[0] == "error"]))
                    nbad += 1
                    continue
                got = po.summary(allres)
                want = po.summary(po.execute(json.dumps(plan), d, world))
                if got != want:
                    failures.append(("fuzz", seed, json.dumps(plan), got, want))
                    nbad += 1
        if rank == 0:
            print("fuzz                   %d plans   oracle    %s (%d bad)" % (a.fuzz, "OK " if not nbad else "BAD", nbad),
                  flush=True)
    # duplicate-key replicated joins (expanding chains) at N ranks vs the reference per node
    for pname in ("dup_build_chain", "dup_probe_chain"):
        d = data(0.01, 42, 1 << 20)
        res = ctx.execute_plan(golden["plans"][pname], d)
        allres = [None] * world
        dist.all_gather_object(allres, (res.schema, res.rows.copy()))
        if rank == 0:
            got = po.summary(allres)
            want = po.summary(po.execute(json.dumps(golden["plans"][pname]), d, world))
            ok = got == want
            print("%-22s dupkeys    oracle    %s rows=%d per_node=%s" % (pname, "OK " if ok else "BAD", got["rows"],
                                                                         got["per_node_rows"]), flush=True)
            if not ok:
                failures.append((pname, "dupkeys", got, want))
    # the distributed-join microbenchmark (run_join variants over NCCL): the union of the ranks'
    # rows equals the reference's run_sim_join rows (tests/golden/join.json)
    jg = json.load(open(os.path.join(ROOT, "tests", "golden", "join.json")))
    for g in jg["joins"][:6]:
        wl = g["workload"]
        for variant in ("blocking", "blocking-opt", "chunking", "deferred"):
            _st, res = ctx.run_synthetic_join(variant, 1 if variant.startswith("blocking") else 2, g["chunk_rows"],
                                              wl["build_rows"], wl["probe_rows"], wl["payload"], wl["hit_ratio"],
                                              wl["seed"])
            allres = [None] * world
            dist.all_gather_object(allres, (res.schema, res.rows.copy()))
            if rank == 0:
                got = po.summary(allres)
                ok = (got["rows"], got["rowhash"], got["colsums"]) == (g["rows"], g["rowhash"], g["colsums"])
                print("%-22s %-10s reference %s rows=%d per_node=%s" % ("join_%d" % wl["seed"], variant,
                                                                       "OK " if ok else "BAD", got["rows"],
                                                                       got["per_node_rows"]), flush=True)
                if not ok:
                    failures.append(("join", variant, wl, got))
    # synthetic-join workload (gen_workload kind=synthetic): per-node rows vs the reference
    syn = json.load(open(os.path.join(ROOT, "tests", "golden", "synthetic.json")))
    sdir = os.path.join(base, "syn")
    if rank == 0:
        psg.gen_workload("synthetic", sdir, devices=world, nodes=world, seed=42, codec="identity")
    dist.barrier()
    for pname in ("syn_agg", "syn_global", "syn_filtered", "syn_noagg"):
        res = ctx.execute_plan(syn["plans"][pname], sdir)
        allres = [None] * world
        dist.all_gather_object(allres, (res.schema, res.rows.copy()))
        if rank == 0:
            got = po.summary(allres)
            g = [r for r in syn["results"] if r["plan"] == pname and r["nodes"] == world and r["seed"] == 42
                 and r["codec"] == "identity"]
            if g:
                want = {k: g[0][k] for k in ("rows", "rowhash", "colsums", "per_node_rows")}
                src = "reference"
            else:
                want = po.summary(po.execute(json.dumps(syn["plans"][pname]), sdir, world))
                src = "oracle"
            ok = all(got[k] == want[k] for k in ("rows", "rowhash", "colsums", "per_node_rows"))
            print("%-22s synthetic  %-9s %s rows=%d per_node=%s" % (pname, src, "OK " if ok else "BAD", got["rows"],
                                                                   got["per_node_rows"]), flush=True)
            if not ok:
                failures.append((pname, "synthetic", got, want))
    # local plans (no shuffle, psg_execute_local): one partial row per rank = per node
    local = json.load(open(os.path.join(ROOT, "tests", "golden", "local.json")))
    for pname in ("q6", "q6_count"):
        d = data(0.1, 42, 1 << 20)
        res = ctx.execute_local(local["plans"][pname], d)
        allres = [None] * world
        dist.all_gather_object(allres, (res.schema, res.rows.copy()))
        if rank == 0:
            g = [r for r in local["results"] if r["plan"] == pname and r["nodes"] == world and r["scale"] == 0.1
                 and r["seed"] == 42 and r["codec"] == "identity"]
            if g:
                want = [(x["rows"], x["colsums"] if x["rows"] else []) for x in g[0]["per_node"]]
                src = "reference"
            else:
                want = [(s["rows"], s["colsums"]) for s in
                        (po.summary([x]) for x in po.execute_local(json.dumps(local["plans"][pname]), d, world))]
                src = "oracle"
            got = [(s["rows"], s["colsums"]) for s in (po.summary([x]) for x in allres)]
            ok = got == want
            print("%-22s local      %-9s %s per_node=%s" % (pname, src, "OK " if ok else "BAD", got), flush=True)
            if not ok:
                failures.append((pname, "local", got, want))
    if rank == 0:
        print("FAILURES", len(failures))
        for f in failures:
            print(f)
    ok = torch.tensor([0 if failures else 1], device="cuda")
    dist.broadcast(ok, src=0)
    ctx.close()
    dist.destroy_process_group()
    sys.exit(0 if ok.item() else 1)


if __name__ == "__main__":
    main()
