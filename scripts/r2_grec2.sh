#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${1:-2}
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for v in "PSG_SLAB_GREC=0" "PSG_SLAB_GREC=1" "PSG_SLAB_GREC=1 PSG_SLAB_DIAG=2" "PSG_SLAB_GREC=0 PSG_SLAB_DIAG=2" "PSG_SLAB_GREC=0 PSG_TMA_NG=3 PSG_TMA_CTAS=1" "PSG_SLAB_GREC=0 PSG_TMA_R=8"; do
  env $v bash -c "$(declare -f tr); N=$N; tr scripts/q3_value_mgpu.py --steps 5 --tag '$v'" 2>&1 | grep '^{' | tail -1
done
PSG_TRACE=1 PSG_SLAB_GREC=1 tr scripts/q3_value_mgpu.py --steps 1 --warmup 0 --tag t 2>&1 | grep "jit kernel" | sort | uniq -c
