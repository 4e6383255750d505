#!/usr/bin/env bash
# Round-2 N=1 evidence at HEAD: gpu tests, smoke, bench line, launch list + ncu of the probe kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_smoke.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err; echo "bench rc=$?"
cat gpurun_out/r2_bench_n1.json; tail -3 gpurun_out/r2_bench_n1.err
timeout 900 bash scripts/profile_n1.sh
