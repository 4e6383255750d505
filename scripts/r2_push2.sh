#!/usr/bin/env bash
# received-rows array (many sub-lists) x push/pull at N=2 and N=4; parity at N=4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tr() { N=$1; shift; timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for N in 2 4; do for v in "PSG_SLAB_PUSH=1 PSG_RECV_SUB=64" "PSG_SLAB_PUSH=1 PSG_RECV_SUB=256" "PSG_SLAB_PUSH=0 PSG_RECV_SUB=64"; do
  env $v bash -c "$(declare -f tr); tr $N scripts/q3_value_mgpu.py --steps 10 --tag 'n$N $v'" 2>&1 | grep -E '^\{|rror' | tail -1
  env $v PSG_TRACE=3 bash -c "$(declare -f tr); tr $N scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag t" 2>&1 | grep -E "slab consume" | tail -1
done; done
PSG_SLAB_PUSH=1 TMO=1500 tr 4 scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu4_parity_push.txt 2>&1
echo "parity4 rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu4_parity_push.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu4_parity_push.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu4_parity_push.txt | head -5
