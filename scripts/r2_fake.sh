#!/usr/bin/env bash
# 1-GPU: the N>1 peer-slab probe kernel profiled in one process (PSG_SLAB_FAKE=1, timing only)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/q3_value.py --tag plain 2>&1 | tail -1
PSG_SLAB_FAKE=1 timeout 300 python scripts/q3_value.py --tag fake 2>&1 | tail -1
PSG_SLAB_FAKE=1 PSG_SLAB_DIAG=2 timeout 300 python scripts/q3_value.py --tag fake_diag2 2>&1 | tail -1
PSG_SLAB_FAKE=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:psg_jit_scan -s 5 -c 1 -o gpurun_out/r2_probe_fake \
  python scripts/q3_value.py --steps 1 --warmup 1 --tag ncu > gpurun_out/r2_ncu_fake.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/r2_ncu_fake.log
