"""Golden fixtures for the distributed-join microbenchmark, from the REFERENCE ITSELF
(oracle/_ref/ref_driver: make_plan, join.cpp:126-134, and run_sim_join, join_harness.cpp:43-97,
all nodes of the join with rows collected). The joined multiset does not depend on the node count
(every probe row meets the same build rows wherever it lands), so GPU runs at any N are checked
against these rowhashes. Development container only."""
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
DRIVER = os.path.join(HERE, "..", "..", "oracle", "_ref", "ref_driver")
VARIANTS = ["blocking", "blocking-opt", "chunking", "deferred"]


def main():
    out = {"schedules": [], "joins": []}
    for v in VARIANTS:
        for streams in (1, 2, 3):
            for lw, rw in ((1, 1), (3, 5), (4, 2), (0, 3), (2, 0), (6, 6)):
                r = subprocess.run([DRIVER, "joinplan", "--variant", v, "--streams", str(streams), "--left", str(lw),
                                    "--right", str(rw)], capture_output=True, text=True)
                if r.returncode != 0:  # blocking variants reject streams != 1 (JoinSpec::validate)
                    continue
                out["schedules"].append({"variant": v, "streams": streams, "left": lw, "right": rw,
                                         "steps": json.loads(r.stdout)})
    workloads = [
        {"build_rows": 120000, "probe_rows": 320000, "payload": 3, "hit_ratio": 0.5, "seed": 42},
        {"build_rows": 50000, "probe_rows": 90000, "payload": 1, "hit_ratio": 1.0, "seed": 7},
        {"build_rows": 1000, "probe_rows": 70000, "payload": 2, "hit_ratio": 0.9, "seed": 3},
        {"build_rows": 0, "probe_rows": 5000, "payload": 1, "hit_ratio": 0.5, "seed": 1},
    ]
    for wl in workloads:
        for v, nodes, chunk in (("deferred", 2, 32768), ("chunking", 4, 10000), ("blocking", 1, 32768)):
            cmd = [DRIVER, "join", "--variant", v, "--nodes", str(nodes), "--streams", "2", "--chunk-rows", str(chunk),
                   "--build-rows", str(wl["build_rows"]), "--probe-rows", str(wl["probe_rows"]), "--payload",
                   str(wl["payload"]), "--hit-ratio", str(wl["hit_ratio"]), "--seed", str(wl["seed"])]
            r = json.loads(subprocess.run(cmd, capture_output=True, text=True, check=True).stdout.strip().splitlines()[-1])
            r.pop("seconds")
            out["joins"].append({"workload": wl, "variant": v, "nodes": nodes, "chunk_rows": chunk, **r})
            print(v, nodes, wl, r["rows"], r["rowhash"])
    with open(os.path.join(HERE, "join.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
