#!/usr/bin/env bash
# N=1: GPU tests, L2 fetch granularity A/B, bench value-loop A/B (clock sampler), launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest9.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest9.log
run() { echo "== $*"; env "$@" timeout 300 python scripts/q3_value.py --tag "$*" 2>&1 | tail -1; }
run PSG_L2_FETCH=0
run PSG_L2_FETCH=32
run PSG_L2_FETCH=64
run PSG_L2_FETCH=128
run PSG_L2_FETCH=32 PSG_TMA=0
run PSG_L2_FETCH=32
PSG_TRACE=3 python scripts/q3_value.py --steps 1 --warmup 2 > gpurun_out/r2_phases_n1.txt 2>&1; tail -14 gpurun_out/r2_phases_n1.txt
python scripts/q3_value.py --steps 2 --warmup 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/r2_launches_n1f.csv \
  python scripts/q3_value.py --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu rc=$?"
PSG_BENCH_VERBOSE=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-block --no-cpu-baseline --budget-gb 0 > gpurun_out/r2_bench_a.json 2> gpurun_out/r2_bench_a.err; echo "bench rc=$?"
PSG_BENCH_NO_CLOCKS=1 PSG_BENCH_VERBOSE=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-block --no-cpu-baseline --budget-gb 0 > gpurun_out/r2_bench_b.json 2> gpurun_out/r2_bench_b.err; echo "bench rc=$?"
for f in a b; do python -c "import json; d=json.loads(open('gpurun_out/r2_bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac'], d['e2e']['value'])"; grep "value steps" gpurun_out/r2_bench_$f.err; done
