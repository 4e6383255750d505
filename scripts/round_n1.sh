#!/usr/bin/env bash
# 1-GPU round-end evidence at HEAD: gpu tests, smoke, bench line (with CPU reference), launch list + probe ncu, phase trace
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/rg_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/rg_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rg_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/rg_smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/rg_bench_n1.json 2> gpurun_out/rg_bench_n1.err; echo "bench rc=$?"
cat gpurun_out/rg_bench_n1.json; tail -3 gpurun_out/rg_bench_n1.err
PSG_TRACE=3 timeout 300 python scripts/q3_value.py --steps 1 --warmup 1 --tag trace > gpurun_out/rg_trace_n1.txt 2>&1
timeout 900 bash scripts/profile_n1.sh
