#!/usr/bin/env bash
# copy-stream callbacks moved off the copy stream (e2e), reduction-mode key-bitmap build; parity
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
timeout 300 python scripts/q3_value.py --tag n1 2>&1 | tail -1
PSG_TIMELINE=gpurun_out/tl_n1b timeout 600 python scripts/timeline_run.py 2>&1 | tail -8
timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --budget-gb 0 2>/dev/null | python -c "
import sys, json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('e2e', d['e2e']['value'], 'block', d['e2e_block']['value'], 'ingest_probe', d['e2e_roofline']['terms']['ingest_pipelined_s'], 'value', d['value'], 'parity', d['parity']['match'], d['parity'].get('block_match'))"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_cb.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_gpu_tests_cb.txt
unset CUDA_VISIBLE_DEVICES
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
tr scripts/q3_value_mgpu.py --steps 10 --tag 'n2' 2>&1 | grep -E '^\{|rror' | tail -1
TMO=1500 tr scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu2_parity_cb.txt 2>&1
echo "parity rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu2_parity_cb.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu2_parity_cb.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu2_parity_cb.txt | head -5
