#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "PSG_BATCH_APPENDS=1" "PSG_BATCH_APPENDS=0" "PSG_SLAB_FAKE=1"; do CUDA_VISIBLE_DEVICES=0 env $v timeout 300 python scripts/q3_value.py --tag "$v" 2>&1 | tail -1; done
CUDA_VISIBLE_DEVICES=0 PSG_SLAB_FAKE=1 PSG_TRACE=3 timeout 300 python scripts/q3_value.py --steps 1 --warmup 1 --tag t 2>&1 | grep "probe side" | tail -1
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for v in "PSG_BATCH_APPENDS=1" "PSG_BATCH_APPENDS=0"; do env $v bash -c "$(declare -f tr); tr scripts/q3_value_mgpu.py --steps 10 --tag '$v'" 2>&1 | grep -E '^\{|rror' | tail -1; done
PSG_TRACE=3 tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag t 2>&1 | grep -E "slab consume|probe \+" | tail -2
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_interp.py tests/test_gpu_q3.py -x -q > gpurun_out/r2_batch_tests.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_batch_tests.txt
