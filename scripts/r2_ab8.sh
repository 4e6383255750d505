#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 300 python scripts/q3_value.py --tag "n1" 2>&1 | tail -1
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for v in "PSG_SLAB_PUSH=0" "PSG_SLAB_PUSH=1" "PSG_CONSUME_BPS=8" "PSG_SLAB_PUSH=1 PSG_CONSUME_BPS=8" "PSG_SLAB_DIAG=4"; do
  env $v bash -c "$(declare -f tr); tr scripts/q3_value_mgpu.py --steps 10 --tag '$v'" 2>&1 | grep -E '^\{|rror' | tail -1
  env $v PSG_TRACE=3 bash -c "$(declare -f tr); tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag t" 2>&1 | grep "slab consume" | tail -1
done
