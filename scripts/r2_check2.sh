#!/usr/bin/env bash
# GPU tests, bucket A/B, launch list, full N=1 bench line (+ out-of-core budget config), box facts.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
df -h /tmp . 2>&1 | tail -3; nproc; free -g | head -2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest6.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest5.log
run() { echo "== $*"; env "$@" timeout 300 python scripts/q3_value.py --tag "$*" 2>&1 | tail -1; }
run PSG_BUCKETS=0
run PSG_BUCKETS=1
run PSG_TMA=0
run PSG_TMA_NG=2 PSG_TMA_NS=4 PSG_TMA_CTAS=2
python scripts/q3_value.py --steps 2 --warmup 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_n1d.csv \
  python scripts/q3_value.py --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_n1c.json 2> gpurun_out/r2_bench_n1c.err; echo "bench rc=$?"
tail -c 4000 gpurun_out/r2_bench_n1c.json
