#!/usr/bin/env bash
# warp-specialised key-bitmap build A/B at N=1 (+ trace), gpu tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in 1 0; do PSG_TMA_KB=$v timeout 300 python scripts/q3_value.py --tag "n1 tma_kb$v" 2>&1 | tail -1; done
PSG_TRACE=3 timeout 300 python scripts/q3_value.py --steps 1 --warmup 1 --tag trace > gpurun_out/r2_trace_n1_kb.txt 2>&1
grep "device\|jit kernel" gpurun_out/r2_trace_n1_kb.txt | tail -16
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_kb.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_gpu_tests_kb.txt
