#!/usr/bin/env bash
# GPU tests + bucketed finalisation A/B at SF100 N=1 + launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest4.log
run() { echo "== $*"; env "$@" timeout 300 python scripts/q3_value.py --tag "$*" 2>&1 | tail -1; }
run PSG_BUCKETS=0
run PSG_BUCKETS=1
run PSG_BUCKETS=1 PSG_TMA=0
run PSG_BUCKETS=1 PSG_TMA_NG=2 PSG_TMA_NS=4 PSG_TMA_CTAS=2
run PSG_BUCKETS=1 PSG_TMA_NG=2 PSG_TMA_NS=5 PSG_TMA_CTAS=2
run PSG_BUCKETS=1 PSG_TMA_NG=1 PSG_TMA_NS=4 PSG_TMA_CTAS=3
run PSG_BUCKETS=0
run PSG_BUCKETS=1
python scripts/q3_value.py --steps 2 --warmup 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_n1b.csv \
  python scripts/q3_value.py --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu rc=$?"
