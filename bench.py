#!/usr/bin/env python
"""Benchmark: TPC-H Q3-analog at SF100, storage-resident, on N B200s (one rank per GPU).

Metric (BASELINE.json): Q3 SF100 query seconds + roofline fraction at 1/2/4/8 B200 vs CPU reference.

  python bench.py [--gpus N --steps K --warmup W]                 # our arm (N>1: under torchrun)
  python bench.py --impl reference --steps K --warmup W           # the reference CPU engine

One "step" = one full query over the SF100 dataset. Two timings per step:
  value : inputs already resident in HBM (psg_stage_plan once, then psg_execute_staged per step);
          device time from CUDA events on the engine's compute stream, max over ranks.
  e2e   : the public call a user makes (psg_execute_plan): PSTO files (page cache) -> pinned ->
          HBM on copy streams -> kernels -> NCCL shuffle -> result rows back to the host.
Data: the reference's generator (byte-identical re-implementation, tests/golden/gen_hashes.json),
seed 42, identity codec, 1 MiB row groups, written once as 8 node shards (dev0..dev7); rank r of N
scans node shards k = r (mod N); customer is replicated. Inputs (24.2 GB) are >> L2 (126 MB).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TPC-H Q3 SF100 query sec + roofline fraction at 1/2/4/8 B200 vs CPU reference"
SHARDS = 8
DATE = 19950315


def plan_for(shards, io_workers):
    o = ["{data}/dev%d/orders.node%d.psto" % (k % SHARDS, k) for k in shards]
    li = ["{data}/dev%d/lineitem.node%d.psto" % ((k + 1) % SHARDS, k) for k in shards]
    return {
        "buffer_target_bytes": 8388608, "io_workers": io_workers,
        "scans": [
            {"table": "customer", "paths": ["{data}/dev0/customer.psto"], "replicated": True,
             "predicate": [{"col": "c_mktsegment", "op": "==", "value": 1}]},
            {"table": "orders", "paths": o, "predicate": [{"col": "o_orderdate", "op": "<", "value": DATE}]},
            {"table": "lineitem", "paths": li, "predicate": [{"col": "l_shipdate", "op": ">", "value": DATE}]}],
        "joins": [
            {"id": "cust_orders", "build": "customer", "probe": "orders", "build_key": "c_custkey",
             "probe_key": "o_custkey", "mode": "replicated"},
            {"id": "result", "build": "cust_orders", "probe": "lineitem", "build_key": "o_orderkey",
             "probe_key": "l_orderkey", "mode": "shuffle"}],
        "aggregate": {"group_by": "l_orderkey", "sums": ["l_extendedprice", "l_discount"]},
    }


def ensure_data(root, scale, nodes, rank_is_writer=True, codec="identity"):
    marker = os.path.join(root, "DONE")
    if os.path.exists(marker):
        return root, 0.0
    if not rank_is_writer:
        return root, 0.0
    import shutil
    import paper_2512_02862_b200 as psg
    shutil.rmtree(root, ignore_errors=True)
    t = time.time()
    psg.gen_workload("tpch", root, devices=nodes, nodes=nodes, scale=scale, seed=42, codec=codec,
                     threads=max(3, min(32, os.cpu_count() or 3)))
    with open(marker, "w") as f:
        f.write(json.dumps({"scale": scale, "nodes": nodes, "seed": 42, "codec": codec}))
    return root, time.time() - t


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
            "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def pinned_h2d_gbs(local, nbytes=1 << 30, reps=3):
    """Pinned host -> HBM copy bandwidth of this GPU's link, measured live (the PCIe term of the
    ingest roofline)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda:%d" % local)
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        t = time.time()
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, nbytes / (time.time() - t) / 1e9)
    del h, d
    return best


def ncu_traffic(scale):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t.get("dram_bytes_per_launch") if float(t.get("scale", -1)) == float(scale) else None
    except Exception:
        return None


# ------------------------------------------------------------------------------ CPU baselines
def cpu_reference_run(sample_scale, steps, warmup, cores, data_dir):
    """Runs the UNMODIFIED reference engine (oracle/_ref/ref_driver, run_socket_pipeline node 0 of 1,
    Overlapped mode) on a bounded sample; returns (per-step seconds list, kind, note)."""
    driver = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    d, _ = ensure_data(os.path.join(data_dir, "sf%g_n1" % sample_scale), sample_scale, 1)
    plan = plan_for([0], cores)
    plan["scans"][1]["paths"] = ["{data}/dev0/orders.node0.psto"]
    plan["scans"][2]["paths"] = ["{data}/dev0/lineitem.node0.psto"]
    if os.path.exists(driver):
        out = subprocess.run([driver, "run", "--plan-json", json.dumps(plan), "--data", d, "--mode", "overlapped",
                              "--backend", "socket", "--repeat", str(steps + warmup)],
                             capture_output=True, text=True, check=True).stdout.strip().splitlines()
        res = [json.loads(x) for x in out if x.startswith("{")]
        return [r["seconds"] for r in res[warmup:]], "reference", res[0]
    # oracle port (numpy restatement), single thread
    from oracle import plan_oracle as po
    times = []
    for i in range(steps + warmup):
        t = time.time()
        r = po.summary(po.execute(json.dumps(plan), d, 1))
        if i >= warmup:
            times.append(time.time() - t)
    return times, "port", r


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    times, kind, r = cpu_reference_run(args.sample_scale, args.steps, args.warmup, cores, args.data_dir)
    scale_up = args.scale / args.sample_scale
    v = statistics.mean(times) * scale_up
    sample = "Q3-analog SF%g (1 node, warm page cache), time x %g extrapolated linearly to SF%g" % (
        args.sample_scale, scale_up, args.scale)
    line = {"metric": METRIC, "impl": "reference", "value": round(v, 4), "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v * 1000, 3), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic (reference generator)",
            "config": {"workload": "Q3-analog SF%g sample of the SF%g query" % (args.sample_scale, args.scale),
                       "engine": "reference execute_plan via run_socket_pipeline (node 0 of 1), Overlapped",
                       "io_workers": cores, "sample_rows": r.get("rows")},
            "cpu_baseline": {"value": round(v, 4), "unit": "s", "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": round(v, 4), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=float, default=100.0)
    ap.add_argument("--sample-scale", type=float, default=10.0)
    ap.add_argument("--data-dir", default=os.environ.get("PSG_BENCH_DATA", "/tmp/psg_bench"))
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-semijoin", action="store_true")
    ap.add_argument("--io-threads", type=int, default=0)
    ap.add_argument("--batch-mb", type=int, default=0,
                    help="ingest batch size; default 128 MB at one GPU, 64 MB per rank at N > 1 (measured: "
                         "bigger batches fill the GPU with inflate work at N=1, smaller ones pipeline better "
                         "when each rank streams 1/N of the data)")
    ap.add_argument("--codec", default="identity", choices=["identity", "block"],
                    help="PSTO codec of the dataset (block = zlib chunks, inflated on the GPU)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import paper_2512_02862_b200 as psg
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cores = os.cpu_count() or 1
    io_threads = args.io_threads or max(2, min(12, cores // max(world, 1)))

    data_root = os.path.join(args.data_dir, "sf%g_n%d%s" % (args.scale, SHARDS, "" if args.codec == "identity"
                                                                  else "_" + args.codec))
    gen_s = 0.0
    if rank == 0:
        data_root, gen_s = ensure_data(data_root, args.scale, SHARDS, codec=args.codec)
    if dist:
        dist.barrier()

    nccl_id = None
    if world > 1:
        obj = [psg.Context.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctx = psg.Context(local, rank, world, nccl_id)
    if not args.batch_mb:
        args.batch_mb = 128 if world == 1 else 64
    ctx.set_ingest(io_threads=io_threads, batch_bytes=args.batch_mb << 20)
    if args.no_semijoin:
        ctx.set_semijoin(False)
    shards = [k for k in range(SHARDS) if k % world == rank]
    plan = plan_for(shards, io_threads)

    def sync_all():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        import torch
        t = torch.tensor([float(x)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if not dist:
            return x
        import torch
        t = torch.tensor([float(x)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())

    # ---------------- value: HBM-resident inputs ----------------
    t = time.time()
    staged = ctx.stage_plan(plan, data_root)
    stage_s = time.time() - t
    for _ in range(args.warmup):
        staged.run(want_rows=False)
    sync_all()
    dev_ms = []
    launches = 0
    probe_ms = probe_bytes = probe_launches = 0
    rows = 0
    clk = Clocks(local).__enter__()
    if True:
        wall0 = time.time()
        for _ in range(args.steps):
            sync_all()  # every step starts aligned across ranks (the barrier is outside the engine's events)
            st = staged.run(want_rows=False)
            dev_ms.append(st["device_ms"])
            launches += st["kernel_launches"]
            probe_ms += st["probe_kernel_ms"]
            probe_bytes += st["probe_kernel_bytes"]
            probe_launches += st["probe_kernel_launches"]
            rows = st["result_rows"]
    sync_all()
    wall_value = (time.time() - wall0) / max(args.steps, 1)
    value_s = max_over_ranks(sum(dev_ms) / 1000.0 / max(args.steps, 1))
    total_groups = sum_over_ranks(rows)
    staged.free()

    # ---------------- e2e: storage-resident, through psg_execute_plan ----------------
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else args.steps
    warm = [ctx.execute_plan(plan, data_root) for _ in range(min(args.warmup, 2))]  # pinned result blocks
    del warm
    sync_all()
    e2e_t, h2d, d2h = [], 0, 0
    e2e_rows = 0
    io_wait = []
    for _ in range(e2e_steps):
        sync_all()
        t = time.time()
        res = ctx.execute_plan(plan, data_root)
        e2e_t.append(time.time() - t)
        h2d, d2h = res.stats["h2d_bytes"], res.stats["result_bytes"]
        io_wait.append(res.stats["io_wait_s"])
        e2e_rows = res.rows.shape[0]
    sync_all()
    clk.__exit__(None, None, None)
    e2e_s = max_over_ranks(statistics.mean(e2e_t)) if e2e_t else None
    h2d_all, d2h_all = sum_over_ranks(h2d), sum_over_ranks(d2h)
    e2e_groups = sum_over_ranks(e2e_rows)

    # ---------------- roofline of the dominant kernel (lineitem fused scan) ----------------
    peak, peak_kind = measured_peak()
    roof = None
    if probe_launches:
        per_launch_bytes = probe_bytes / probe_launches
        per_launch_s = probe_ms / 1000.0 / probe_launches
        achieved = per_launch_bytes / per_launch_s / 1e9
        ach = max_over_ranks(-achieved) * -1 if dist else achieved  # slowest rank
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": ncu_traffic(args.scale), "kernel": "psg_jit_scan SINK_PROBE (lineitem scan+filter+probe+agg)"
                if world == 1 else "k_scan<4,SINK_MATERIALIZE> (lineitem scan+filter+partition)",
                "algorithmic_bytes_per_launch": int(per_launch_bytes), "peak_kind": peak_kind,
                "kernel_ms_per_launch": round(per_launch_s * 1000, 4),
                "share_of_step": round(probe_ms / max(sum(dev_ms), 1e-9), 4)}

    # binding roofline of the end-to-end query: ingest (per-GPU bytes over the pinned->HBM link),
    # the slowest rank decides; the host's page-cache read bandwidth is shared by all ranks and is
    # the tighter bound on this box (profiles/r1_box_ingest_probe.txt)
    e2e_roof = None
    try:
        bw = pinned_h2d_gbs(local)
        t_min = max_over_ranks(h2d / 1e9 / bw) if bw > 0 else None
        if t_min and e2e_s:
            e2e_roof = {"bound": "ingest (pinned H2D per GPU)", "h2d_gbs_measured": round(bw, 1),
                        "t_min_s": round(t_min, 4), "frac": round(t_min / e2e_s, 4)}
    except Exception as e:  # never hide the main numbers
        e2e_roof = {"error": str(e)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            times, kind, r = cpu_reference_run(args.sample_scale, 1, 0, cores, args.data_dir)
            f = args.scale / args.sample_scale
            cpu = {"value": round(statistics.mean(times) * f, 3), "unit": "s", "cores": cores, "kind": kind,
                   "sample": "Q3-analog SF%g (node 0 of 1, Overlapped, warm page cache, io_workers=%d) x %g "
                             "extrapolated linearly to SF%g" % (args.sample_scale, cores, f, args.scale)}
        except Exception as e:  # baseline failure must not hide the GPU number
            cpu = {"value": None, "unit": "s", "cores": cores, "kind": "reference", "sample": "failed: %s" % e}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value_s, 6), "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(value_s * 1000, 4), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic: reference TPC-H-analog generator, seed 42 (byte-identical re-implementation)",
            "config": {"workload": "Q3-analog SF%g canonical plan (o_orderdate<%d, l_shipdate>%d, group by l_orderkey)"
                                   % (args.scale, DATE, DATE),
                       "scale": args.scale, "row_group_bytes": 1 << 20, "codec": args.codec,
                       "layout": "8 node shards; rank r scans shards k%%N==r; customer replicated",
                       "l2": "inputs 24.2 GB >> 126 MB L2 (no flush needed)",
                       "value": "HBM-resident inputs, CUDA events on the engine stream, max over ranks",
                       "io_threads": io_threads, "batch_mb": args.batch_mb,
                       "semijoin_bloom": not args.no_semijoin, "stage_s": round(stage_s, 3),
                       "gen_s": round(gen_s, 2), "groups": int(total_groups), "wall_s_per_value_step": round(wall_value, 6)},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_s, 4) if e2e_s else None, "unit": "s", "h2d_bytes_per_step": int(h2d_all),
                    "d2h_bytes_per_step": int(d2h_all), "steps": e2e_steps, "groups": int(e2e_groups),
                    "io_wait_s": round(statistics.mean(io_wait), 4) if io_wait else None,
                    "ingest_gbs": round(h2d_all / 1e9 / e2e_s, 2) if e2e_s else None,
                    "path": "psg_execute_plan: PSTO files (warm page cache) -> pinned -> HBM -> rows to host"},
            "e2e_roofline": e2e_roof,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
