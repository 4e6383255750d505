#!/usr/bin/env bash
# global records (one lookup per probe row at N>1): N=1 check, N=2 value + trace + parity
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${1:-2}
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
CUDA_VISIBLE_DEVICES=0 timeout 300 python scripts/q3_value.py --tag "n1" 2>&1 | tail -1
tr scripts/q3_value_mgpu.py --steps 10 --tag 'n2' 2>&1 | grep '^{' | tail -1
PSG_SLAB_DIAG=2 tr scripts/q3_value_mgpu.py --steps 5 --tag 'n2 diag2' 2>&1 | grep '^{' | tail -1
PSG_TRACE=3 tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace > gpurun_out/r2_trace_n${N}_grec.txt 2>&1
grep "device\|jit kernel" gpurun_out/r2_trace_n${N}_grec.txt | tail -20
TMO=1500 tr scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu${N}_parity_grec.txt 2>&1
echo "parity rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu${N}_parity_grec.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu${N}_parity_grec.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu${N}_parity_grec.txt | head -5
