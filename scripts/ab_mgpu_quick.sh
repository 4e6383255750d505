#!/usr/bin/env bash
# Quick knob A/B at N GPUs: staged SF100 query median/mean per variant (no traces)
#   bash scripts/ab_mgpu_quick.sh N "PSG_X=0" "PSG_X=1" ...
cd "$(dirname "$0")/.."
N=$1; shift
for v in "$@"; do
  echo "$v: $(env $v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 1000)) scripts/q3_value_mgpu.py --steps 20 2>&1 | grep -E '^\{' | cut -c1-150)"
done
