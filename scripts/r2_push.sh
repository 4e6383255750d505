#!/usr/bin/env bash
cd "$(dirname "$0")/.."
tr() { N=$1; shift; timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for N in 2 4; do for v in "PSG_SLAB_PUSH=0" "PSG_SLAB_PUSH=1"; do
  env $v bash -c "$(declare -f tr); tr $N scripts/q3_value_mgpu.py --steps 10 --tag 'n$N $v'" 2>&1 | grep -E '^\{|rror' | tail -1
  env $v PSG_TRACE=3 bash -c "$(declare -f tr); tr $N scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag t" 2>&1 | grep -E "slab consume|probe \+" | tail -2
done; done
