#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 PSG_SLAB_FAKE=1 timeout 300 python scripts/q3_value.py --tag fake 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_interp.py -x -q -k slab > gpurun_out/r2_tp_test.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2_tp_test.txt
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
tr scripts/q3_value_mgpu.py --steps 10 --tag 'n2' 2>&1 | grep -E '^\{|rror' | tail -1
PSG_TRACE=3 tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag t 2>&1 | grep -E "slab consume|probe \+" | tail -2
TMO=1500 tr scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu2_parity_tp.txt 2>&1
echo "parity rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu2_parity_tp.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu2_parity_tp.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu2_parity_tp.txt | head -5
