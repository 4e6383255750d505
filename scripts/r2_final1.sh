#!/usr/bin/env bash
# 1-GPU evidence at HEAD: smoke, bench line (with CPU reference), reference arm, launch list + probe ncu, phase trace
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/rf_smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/rf_bench_n1.json 2> gpurun_out/rf_bench_n1.err; echo "bench rc=$?"
cat gpurun_out/rf_bench_n1.json; tail -3 gpurun_out/rf_bench_n1.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/rf_ref.json 2> gpurun_out/rf_ref.err; echo "ref rc=$?"; cat gpurun_out/rf_ref.json | cut -c1-600
PSG_TRACE=3 timeout 300 python scripts/q3_value.py --steps 1 --warmup 1 --tag trace > gpurun_out/rf_trace_n1.txt 2>&1
timeout 900 bash scripts/profile_n1.sh
