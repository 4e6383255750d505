#!/usr/bin/env bash
# bucket sub-lists A/B (PSG_BUCKET_SUB) at N=1 and N=2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${1:-2}
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for s in 1 4 16 32; do CUDA_VISIBLE_DEVICES=0 PSG_BUCKET_SUB=$s timeout 300 python scripts/q3_value.py --tag "n1 sub$s" 2>&1 | tail -1; done
for s in 1 16 32; do PSG_BUCKET_SUB=$s bash -c "$(declare -f tr); N=$N; tr scripts/q3_value_mgpu.py --steps 5 --tag 'n2 sub$s'" 2>&1 | grep '^{' | tail -1; done
PSG_TRACE=3 tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace > gpurun_out/r2_trace_n${N}_sub.txt 2>&1
grep device gpurun_out/r2_trace_n${N}_sub.txt | tail -16
