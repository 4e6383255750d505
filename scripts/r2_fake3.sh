#!/usr/bin/env bash
# gpu tests (deferred local-table flags) + fake-slab v3 timing and ncu
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_lt.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_gpu_tests_lt.txt
timeout 300 python scripts/q3_value.py --tag plain 2>&1 | tail -1
PSG_SLAB_FAKE=1 timeout 300 python scripts/q3_value.py --tag fake3 2>&1 | tail -1
PSG_SLAB_FAKE=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:psg_jit_scan -s 5 -c 1 -o gpurun_out/r2_probe_fake3 \
  python scripts/q3_value.py --steps 1 --warmup 1 --tag ncu > gpurun_out/r2_ncu_fake3.log 2>&1; echo "ncu rc=$?"
PSG_JIT_DUMP=gpurun_out PSG_SLAB_FAKE=1 timeout 300 python scripts/q3_value.py --steps 1 --warmup 0 --tag dump > /dev/null 2>&1; ls gpurun_out/psg_jit_* | head
