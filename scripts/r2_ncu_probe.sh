#!/usr/bin/env bash
# ncu --set full of the SF100 N=1 probe kernel (3rd psg_jit_scan launch of the first query):
# staged (bulk-copy) variant and the register-only variant (PSG_TMA=0).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/q3_value.py --steps 1 --warmup 0 --tag plain > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:psg_jit_scan -s 2 -c 1 -o gpurun_out/r2_probe_staged \
  python scripts/q3_value.py --steps 1 --warmup 0 --tag ncu > gpurun_out/ncu_staged.log 2>&1
echo "ncu staged rc=$?"
PSG_TMA=0 python scripts/q3_value.py --steps 1 --warmup 0 --tag plain0 >> gpurun_out/ncu_plain.log 2>&1 && \
PSG_TMA=0 ncu --set full --clock-control none --import-source on -k regex:psg_jit_scan -s 2 -c 1 -o gpurun_out/r2_probe_regs \
  python scripts/q3_value.py --steps 1 --warmup 0 --tag ncu0 > gpurun_out/ncu_regs.log 2>&1
echo "ncu regs rc=$?"
tail -2 gpurun_out/ncu_plain.log
