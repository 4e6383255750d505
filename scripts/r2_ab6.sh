#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES_ALL=0,1
for v in "PSG_JIT_R=p" "PSG_JIT_R=pk"; do CUDA_VISIBLE_DEVICES=0 env $v timeout 300 python scripts/q3_value.py --tag "n1 $v" 2>&1 | tail -1; done
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bucket_emit -s 1 -c 1 -o gpurun_out/r2_emit \
  python scripts/q3_value.py --steps 1 --warmup 1 --tag ncu > gpurun_out/r2_ncu_emit.log 2>&1; echo "ncu rc=$?"
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
tr scripts/q3_value_mgpu.py --steps 10 --tag 'n2 v3' 2>&1 | grep -E '^\{|rror' | tail -1
PSG_TRACE=1 tr scripts/q3_value_mgpu.py --steps 1 --warmup 0 --tag t 2>&1 | grep "jit kernel" | sort | uniq -c
PSG_TRACE=3 tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace > gpurun_out/r2_trace_n2_v3.txt 2>&1; grep device gpurun_out/r2_trace_n2_v3.txt | tail -15
