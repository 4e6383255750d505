#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "PSG_BUILD_KEY_EARLY=0" "PSG_BUILD_KEY_EARLY=1" "PSG_JIT_MINB=8" "PSG_JIT_MINB=4"; do CUDA_VISIBLE_DEVICES=0 env $v timeout 300 python scripts/q3_value.py --tag "$v" 2>&1 | tail -1; done
CUDA_VISIBLE_DEVICES=0 PSG_BUILD_KEY_EARLY=1 PSG_TRACE=3 timeout 300 python scripts/q3_value.py --steps 1 --warmup 1 --tag trace 2>&1 | grep "build side scan" | tail -1
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for s in 1 4 8 16; do PSG_BUCKET_SUB=$s bash -c "$(declare -f tr); tr scripts/q3_value_mgpu.py --steps 10 --tag 'n2 sub$s'" 2>&1 | grep -E '^\{|rror' | tail -1; done
