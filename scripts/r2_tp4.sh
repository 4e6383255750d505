#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tr() { N=$1; shift; timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for v in "PSG_TILE_PUT=1" "PSG_TILE_PUT=0"; do env $v bash -c "$(declare -f tr); tr 4 scripts/q3_value_mgpu.py --steps 10 --tag 'n4 $v'" 2>&1 | grep -E '^\{|rror' | tail -1; done
TMO=1500 tr 4 scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu4_parity_tp.txt 2>&1
echo "parity4 rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu4_parity_tp.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu4_parity_tp.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu4_parity_tp.txt | head -5
PSG_TRACE=3 tr 4 scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag t 2>&1 | grep device | tail -14
