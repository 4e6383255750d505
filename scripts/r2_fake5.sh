#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PSG_SLAB_FAKE=1 timeout 300 python scripts/q3_value.py --tag fake 2>&1 | tail -1
PSG_SLAB_FAKE=1 PSG_SLAB_DIAG=2 timeout 300 python scripts/q3_value.py --tag fake_diag2 2>&1 | tail -1
PSG_SLAB_FAKE=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:psg_jit_scan -s 5 -c 1 -o gpurun_out/r2_probe_fake5 \
  python scripts/q3_value.py --steps 1 --warmup 1 --tag ncu > gpurun_out/r2_ncu_fake5.log 2>&1; echo "ncu rc=$?"
