#!/usr/bin/env bash
# 2-GPU box: where the peer-slab probe's time goes (PSG_SLAB_DIAG variants are timing-only).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${1:-2}
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for v in "PSG_SLAB=1" "PSG_SLAB_DIAG=1" "PSG_SLAB_DIAG=2" "PSG_SLAB_DIAG=4" "PSG_SLAB_DIAG=6" "PSG_TMA=0" "PSG_SLAB=0" "PSG_SLAB=0 PSG_TMA=0"; do
  echo "== $v"; env $v bash -c "$(declare -f tr); N=$N; tr scripts/q3_value_mgpu.py --steps 5 --tag '$v'" 2>&1 | grep '^{' | tail -1
done
PSG_TRACE=3 PSG_SLAB_DIAG=6 tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace > gpurun_out/r2_trace_n${N}_diag6.txt 2>&1
grep device gpurun_out/r2_trace_n${N}_diag6.txt | tail -16
