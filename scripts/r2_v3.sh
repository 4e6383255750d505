#!/usr/bin/env bash
# branch-free slab probe (v3) vs v2: fake timing at N=1, N=2 values, parity
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in 3 2; do PSG_SLAB_V=$v PSG_SLAB_FAKE=1 timeout 300 python scripts/q3_value.py --tag "fake v$v" 2>&1 | tail -1; done
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for v in 3 2; do PSG_SLAB_V=$v bash -c "$(declare -f tr); tr scripts/q3_value_mgpu.py --steps 10 --tag 'n2 v$v'" 2>&1 | grep -E '^\{|rror' | tail -1; done
PSG_TRACE=1 tr scripts/q3_value_mgpu.py --steps 1 --warmup 0 --tag t 2>&1 | grep "jit kernel" | sort | uniq -c
TMO=1500 tr scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu2_parity_v3.txt 2>&1
echo "parity rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu2_parity_v3.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu2_parity_v3.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu2_parity_v3.txt | head -5
