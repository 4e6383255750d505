#!/usr/bin/env bash
# GPU tests (incl. the join microbenchmark) + staged-kernel shape A/B (rows per lane, groups) at
# SF100 N=1 + the join microbenchmark at N=1.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest7.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest7.log
run() { echo "== $*"; env "$@" timeout 300 python scripts/q3_value.py --tag "$*" 2>&1 | tail -1; }
run PSG_TMA=0
run PSG_TMA=1
run PSG_TMA_R=8 PSG_TMA_NG=2 PSG_TMA_NS=4 PSG_TMA_CTAS=2
run PSG_TMA_R=8 PSG_TMA_NG=4 PSG_TMA_NS=6 PSG_TMA_CTAS=2
run PSG_TMA_R=8 PSG_TMA_NG=3 PSG_TMA_NS=4 PSG_TMA_CTAS=2
run PSG_TMA_R=8 PSG_TMA_NG=6 PSG_TMA_NS=8 PSG_TMA_CTAS=1
run PSG_TMA_R=4 PSG_TMA_NG=2 PSG_TMA_NS=4 PSG_TMA_CTAS=2
run PSG_TMA=1
run PSG_TMA_MAT=1 PSG_TMA_NS=4
echo "== with nvidia-smi polling (bench's clock sampler)"
(nvidia-smi --query-gpu=clocks.sm --format=csv,noheader -lms 100 > /dev/null 2>&1 & echo $! > /tmp/smi.pid)
run PSG_TMA=1
kill $(cat /tmp/smi.pid)
python scripts/q3_value.py --steps 2 --warmup 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_n1e.csv \
  python scripts/q3_value.py --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 python scripts/join_bench.py --build-rows 120000000 --probe-rows 320000000 > gpurun_out/r2_join_n1.json 2> gpurun_out/r2_join_n1.err; echo "join rc=$?"
cat gpurun_out/r2_join_n1.json; tail -3 gpurun_out/r2_join_n1.err
