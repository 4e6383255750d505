#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for v in "PSG_CONSUME_PREFETCH=0" "PSG_CONSUME_PREFETCH=2" "PSG_CONSUME_PREFETCH=1"; do
  env $v bash -c "$(declare -f tr); tr scripts/q3_value_mgpu.py --steps 10 --tag '$v'" 2>&1 | grep -E '^\{|rror' | tail -1
  env $v PSG_TRACE=3 bash -c "$(declare -f tr); tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag t" 2>&1 | grep -E "slab consume|barrier|probe \+" | tail -3
done
