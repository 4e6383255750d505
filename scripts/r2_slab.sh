#!/usr/bin/env bash
# 2-GPU box: key-bitmap build + peer-slab shuffle. N=1 value/parity, N=2 parity (random plans,
# SF10), N=2 value with/without the slab path, phase traces, gpu tests, N=2 bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${1:-2}
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
CUDA_VISIBLE_DEVICES=0 timeout 300 python scripts/q3_value.py --tag n1 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 PSG_KEYBITS=0 timeout 300 python scripts/q3_value.py --tag n1_nokb 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 PSG_TRACE=3 timeout 300 python scripts/q3_value.py --steps 1 --warmup 1 --tag trace1 > gpurun_out/r2_trace_n1c.txt 2>&1
tr scripts/q3_value_mgpu.py --tag slab 2>&1 | grep -E '^\{|Error|error' | tail -3
PSG_SLAB=0 tr scripts/q3_value_mgpu.py --tag noslab 2>&1 | grep '^{' | tail -1
PSG_TRACE=3 tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace > gpurun_out/r2_trace_n${N}b.txt 2>&1
TMO=1500 tr scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu${N}_parity_slab.txt 2>&1
echo "parity rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu${N}_parity_slab.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu${N}_parity_slab.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu${N}_parity_slab.txt | head -5
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_slab.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_gpu_tests_slab.txt
TMO=1200 tr bench.py --gpus $N --steps 10 --warmup 3 --no-block > gpurun_out/r2_bench_n${N}_slab.json 2> gpurun_out/r2_bench_n${N}_slab.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench_n${N}_slab.json; tail -3 gpurun_out/r2_bench_n${N}_slab.err
