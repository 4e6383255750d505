#!/usr/bin/env bash
# join microbenchmark at N=1 (big workload), ncu of the bucket emit and the staged probe.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_join.py tests/test_gpu_q3.py -x -q > gpurun_out/r2_pytest8.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest8.log
timeout 900 python scripts/join_bench.py --build-rows 120000000 --probe-rows 320000000 > gpurun_out/r2_join_n1.json 2> gpurun_out/r2_join_n1.err; echo "join rc=$?"
cat gpurun_out/r2_join_n1.json; tail -3 gpurun_out/r2_join_n1.err
python scripts/q3_value.py --steps 1 --warmup 0 --tag plain > gpurun_out/ncu3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bucket_emit|psg_jit_scan" -s 2 -c 2 -o gpurun_out/r2_probe_emit \
  python scripts/q3_value.py --steps 1 --warmup 0 --tag ncu > gpurun_out/ncu3.log 2>&1; echo "ncu rc=$?"
