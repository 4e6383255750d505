"""SF100 golden result of the bench workload, from the REFERENCE ITSELF.

The bench (bench.py) scans the reference generator's SF100 dataset written as 8 node shards
(seed 42, identity codec, 1 MiB row groups); rank r of N scans shards k = r (mod N). The union over
ranks is the full SF100 Q3-analog query, so its result equals the reference engine's run over all
8 shards as node 0 of 1 (execute_plan via run_socket_pipeline, pipeline_harness.cpp:81-109):
    python tests/golden/make_golden_sf100.py [data_root]
writes sf100.json (groups, rowhash, column sums). rowhash is additive over ranks, so the GPU
bench checks sum_r rowhash_r against it. Development container only (needs oracle/_ref)."""
import json
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def main():
    import bench
    data = sys.argv[1] if len(sys.argv) > 1 else "/tmp/psg_bench/sf100_n8"
    bench.gen_data_subprocess(data, 100.0, bench.SHARDS, "identity")
    plan = bench.plan_for(range(bench.SHARDS), os.cpu_count() or 8)
    t = time.time()
    r = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_driver"), "run", "--plan-json", json.dumps(plan),
                        "--data", data, "--mode", "overlapped", "--backend", "socket", "--repeat", "1"],
                       capture_output=True, text=True, check=True)
    res = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][0])
    out = {"workload": "Q3-analog SF100 canonical plan (bench.plan_for over 8 node shards, node 0 of 1)",
           "scale": 100.0, "shards": bench.SHARDS, "seed": 42, "codec": "identity", "row_group_bytes": 1 << 20,
           "plan": plan, "groups": res["rows"], "rowhash": res["rowhash"], "colsums": res["colsums"],
           "schema": ["l_orderkey", "rows", "sum_l_extendedprice", "sum_l_discount"],
           "reference_seconds": res["seconds"], "reference_cores": os.cpu_count(),
           "generated_by": "oracle/_ref/ref_driver run (unmodified reference, run_socket_pipeline node 0 of 1, "
                           "Overlapped)", "wall_s": round(time.time() - t, 1)}
    with open(os.path.join(HERE, "sf100.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out)[:400])


if __name__ == "__main__":
    main()
