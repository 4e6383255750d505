#!/usr/bin/env bash
# A/B of engine knobs at N GPUs (torchrun; SF100 HBM-resident query, summed-rowhash parity) with
# the phase trace of the peer-slab probe and fold:
#   bash scripts/ab_mgpu.sh N "PSG_X=0" "PSG_X=1" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=$1; shift
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for v in "$@"; do
  env $v bash -c "$(declare -f tr); N=$N; tr scripts/q3_value_mgpu.py --steps 10 --tag '$v'" 2>&1 | grep -E '^\{|rror' | tail -1
  env $v PSG_TRACE=3 bash -c "$(declare -f tr); N=$N; tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag t" 2>&1 | grep -E "slab consume|probe \+" | tail -2
done
