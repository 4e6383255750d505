#!/usr/bin/env bash
# 2-GPU box: phase breakdowns (PSG_TRACE=3, device time per phase, no syncs) at N=1 and N=2, N=2
# value, bench line and multi-GPU parity.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${1:-2}
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
CUDA_VISIBLE_DEVICES=0 PSG_TRACE=3 timeout 300 python scripts/q3_value.py --steps 1 --warmup 1 --tag trace1 > gpurun_out/r2_trace_n1.txt 2>&1
PSG_TRACE=3 tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace > gpurun_out/r2_trace_n${N}.txt 2>&1
tr scripts/q3_value_mgpu.py --tag plain 2>&1 | grep '^{' | tail -1
TMO=1200 tr bench.py --gpus $N --steps 10 --warmup 3 --no-block > gpurun_out/r2_bench_n${N}.json 2> gpurun_out/r2_bench_n${N}.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench_n${N}.json
TMO=1500 tr scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu${N}_parity.txt 2>&1
echo "parity rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu${N}_parity.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu${N}_parity.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu${N}_parity.txt | head -5
