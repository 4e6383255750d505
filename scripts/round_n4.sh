#!/usr/bin/env bash
# Round-end 4-GPU check: the fallback parity tests, then scripts/final_check.sh (smoke, N=2/4
# parity incl. random plans and SF10, bench refresh at N=1/2/4).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_interp.py tests/test_gpu_multi.py -q > gpurun_out/pytest_fallbacks.log 2>&1
echo "fallback+multi pytest rc=$?"; tail -2 gpurun_out/pytest_fallbacks.log
bash scripts/final_check.sh
