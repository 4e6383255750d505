#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_interp.py -x -q -k "slab or rank_table" > gpurun_out/r2_fake_test.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_fake_test.txt
PSG_SLAB_FAKE=1 timeout 300 python scripts/q3_value.py --tag fake 2>&1 | tail -1
PSG_SLAB_FAKE=1 PSG_TRACE=3 timeout 300 python scripts/q3_value.py --steps 1 --warmup 1 --tag t 2>&1 | grep device | tail -6
PSG_SLAB_FAKE=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_slab_consume -s 1 -c 1 -o gpurun_out/r2_consume \
  python scripts/q3_value.py --steps 1 --warmup 1 --tag ncu > gpurun_out/r2_ncu_consume.log 2>&1; echo "ncu rc=$?"
