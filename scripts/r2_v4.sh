#!/usr/bin/env bash
# screen-first probes: N=1 (PSG_RANK_SCREEN) and fake slab v4 vs v3; N=2 v4 vs v3 + parity
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "PSG_RANK_SCREEN=0" "PSG_RANK_SCREEN=1" "PSG_SLAB_FAKE=1 PSG_SLAB_V=3" "PSG_SLAB_FAKE=1 PSG_SLAB_V=4"; do
  CUDA_VISIBLE_DEVICES=0 env $v timeout 300 python scripts/q3_value.py --tag "$v" 2>&1 | tail -1; done
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for v in 4 3; do PSG_SLAB_V=$v bash -c "$(declare -f tr); tr scripts/q3_value_mgpu.py --steps 10 --tag 'n2 v$v'" 2>&1 | grep -E '^\{|rror' | tail -1; done
TMO=1500 tr scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu2_parity_v4.txt 2>&1
echo "parity rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu2_parity_v4.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu2_parity_v4.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu2_parity_v4.txt | head -5
