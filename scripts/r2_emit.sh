#!/usr/bin/env bash
# warp look-back + 4-way fold in the bucket emit: N=1 value, parity, emit ncu; N=2 value
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 300 python scripts/q3_value.py --tag "n1" 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bucket_emit -s 1 -c 1 -o gpurun_out/r2_emit2 \
  python scripts/q3_value.py --steps 1 --warmup 1 --tag ncu > gpurun_out/r2_ncu_emit2.log 2>&1; echo "ncu rc=$?"
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
tr scripts/q3_value_mgpu.py --steps 10 --tag 'n2' 2>&1 | grep -E '^\{|rror' | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_q3.py tests/test_gpu_interp.py tests/test_gpu_synthetic.py -x -q > gpurun_out/r2_tests_emit.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_tests_emit.txt
