#!/usr/bin/env bash
# NVLink OR of the rank key bitmaps (k_or_own) at N=2: value A/B, trace, parity
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for v in 1 0; do PSG_KB_OR=$v bash -c "$(declare -f tr); tr scripts/q3_value_mgpu.py --steps 10 --tag 'n2 or$v'" 2>&1 | grep -E '^\{|rror' | tail -1; done
PSG_TRACE=3 tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace > gpurun_out/r2_trace_n2_or.txt 2>&1; grep device gpurun_out/r2_trace_n2_or.txt | tail -15
TMO=1500 tr scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu2_parity_or.txt 2>&1
echo "parity rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu2_parity_or.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu2_parity_or.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu2_parity_or.txt | head -5
