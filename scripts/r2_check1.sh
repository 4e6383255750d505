#!/usr/bin/env bash
# Round-2 first GPU check: gpu tests, N=1 bench (short), reference arm (short budget).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench_n1.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 --ref-budget-s 500 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo "ref rc=$?"
cat gpurun_out/r2_ref.json
nproc; free -g | head -2
