#!/usr/bin/env bash
# A/B of the warp-specialised bulk-copy probe (PSG_TMA) and its shape knobs at SF100, N=1.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest2.log
run() { echo "== $*"; env "$@" timeout 300 python scripts/q3_value.py --tag "$*" 2>&1 | tail -2; }
run PSG_TMA=0
run PSG_TMA=1
run PSG_TMA_NG=1 PSG_TMA_NS=4 PSG_TMA_CTAS=3
run PSG_TMA_NG=2 PSG_TMA_NS=4 PSG_TMA_CTAS=2
run PSG_TMA_NG=3 PSG_TMA_NS=6 PSG_TMA_CTAS=1
run PSG_TMA_NG=3 PSG_TMA_NS=9 PSG_TMA_CTAS=1
run PSG_TMA_NG=1 PSG_TMA_NS=3 PSG_TMA_CTAS=4
run PSG_TMA=0
run PSG_TMA=1
