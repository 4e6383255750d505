#!/usr/bin/env bash
cd "$(dirname "$0")/.."
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for v in "PSG_SLAB_DIAG=0" "PSG_SLAB_DIAG=16" "PSG_SLAB_DIAG=20"; do
  env $v PSG_TRACE=3 bash -c "$(declare -f tr); tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag t" 2>&1 | grep -E "slab consume" | tail -1
done
