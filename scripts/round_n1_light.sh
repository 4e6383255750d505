#!/usr/bin/env bash
# 1-GPU round-end evidence without the ncu --set full capture (scripts/round_n1.sh has it): gpu
# tests, smoke, bench line, launch list of one staged query, phase trace
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/rg_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/rg_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rg_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/rg_smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/rg_bench_n1.json 2> gpurun_out/rg_bench_n1.err; echo "bench rc=$?"
tail -1 gpurun_out/rg_bench_n1.json | cut -c1-300
PSG_TRACE=3 timeout 300 python scripts/q3_value.py --steps 1 --warmup 1 --tag trace 2>&1 | grep -E "device .* ms" | tail -12 > gpurun_out/rg_trace_n1.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv \
  python scripts/profile_q3.py --warmup 1 --steps 1 > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_n1.csv $(( $(grep -c gpu__time_duration gpurun_out/launches_n1.csv) / 2 )) > gpurun_out/rg_launches_n1.txt 2>&1
tail -25 gpurun_out/rg_launches_n1.txt
