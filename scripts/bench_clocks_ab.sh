#!/usr/bin/env bash
# The nvidia-smi clock sampler's effect on the staged N-GPU query (median / mean / max device ms):
# off, one sampler for the job at 100 ms, at 500 ms
#   bash scripts/bench_clocks_ab.sh N
cd "$(dirname "$0")/.."
N=${1:-4}
tr() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for rep in 1 2; do
  echo "off: $(tr scripts/q3_value_mgpu.py --steps 30 2>&1 | grep -E '^\{' | cut -c1-120)"
  echo "one sampler 100ms: $(tr scripts/q3_value_mgpu.py --steps 30 --clocks 2>&1 | grep -E '^\{' | cut -c1-120)"
  echo "one sampler 500ms: $(PSG_CLOCKS_MS=500 tr scripts/q3_value_mgpu.py --steps 30 --clocks 2>&1 | grep -E '^\{' | cut -c1-120)"
done
