#!/usr/bin/env bash
# Phase trace (PSG_TRACE=3: device time per phase from CUDA events) of one staged SF100 query at N GPUs
#   bash scripts/trace_mgpu.sh N [ENV=VALUE ...]
cd "$(dirname "$0")/.."
N=$1; shift
env "$@" PSG_TRACE=3 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port $((29500 + RANDOM % 1000)) scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace 2>&1 | grep -E "device .* ms"
