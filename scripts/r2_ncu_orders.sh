#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/q3_value.py --tag n1 2>&1 | tail -1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:psg_jit_scan -s 4 -c 1 -o gpurun_out/r2_orders \
  python scripts/q3_value.py --steps 1 --warmup 1 --tag ncu > gpurun_out/r2_ncu_orders.log 2>&1; echo "ncu rc=$?"
PSG_JIT_DUMP=gpurun_out timeout 300 python scripts/q3_value.py --steps 1 --warmup 0 --tag dump > /dev/null 2>&1; ls gpurun_out/psg_jit_*.cu | tail -3
