#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/q3_value.py --tag n1 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bucket_emit -c 3 python scripts/q3_value.py --steps 1 --warmup 1 --tag ncu 2>&1 | grep -E "k_bucket_emit|gpu__time" | head -6
timeout 900 python -m pytest tests/test_gpu_q3.py tests/test_gpu_interp.py tests/test_gpu_fuzz.py -x -q > gpurun_out/r2_pemit_tests.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2_pemit_tests.txt
