#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
tr scripts/q3_value_mgpu.py --steps 10 --tag 'n2' 2>&1 | grep -E '^\{|rror' | tail -1
PSG_TRACE=3 tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag t 2>&1 | grep device | tail -14
TMO=1500 tr scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu2_parity_ag.txt 2>&1
echo "parity rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu2_parity_ag.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu2_parity_ag.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu2_parity_ag.txt | head -5
