#!/usr/bin/env bash
# 4-GPU box: parity at N=4 and N=2 (random plans + SF10), values at N=2/4, bench line at N=4,
# single-pass ncu DRAM bytes of rank 0's kernels at N=4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tr() { N=$1; shift; timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
TMO=1500 tr 4 scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu4_parity.txt 2>&1
echo "parity4 rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu4_parity.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu4_parity.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu4_parity.txt | head -5
tr 4 scripts/q3_value_mgpu.py --steps 10 --tag n4 2>&1 | grep '^{' | tail -1
PSG_SLAB=0 tr 4 scripts/q3_value_mgpu.py --steps 10 --tag n4_noslab 2>&1 | grep '^{' | tail -1
tr 2 scripts/q3_value_mgpu.py --steps 10 --tag n2 2>&1 | grep '^{' | tail -1
PSG_TRACE=3 tr 4 scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace > gpurun_out/r2_trace_n4.txt 2>&1
grep "device" gpurun_out/r2_trace_n4.txt | tail -16
tr 4 --no-python scripts/ncu_rank0.sh scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag ncu > gpurun_out/r2_ncu_rank0_n4.log 2>&1; echo "ncu rc=$?"
TMO=1200 tr 4 bench.py --gpus 4 --steps 10 --warmup 3 --no-block > gpurun_out/r2_bench_n4.json 2> gpurun_out/r2_bench_n4.err; echo "bench4 rc=$?"
tail -c 2500 gpurun_out/r2_bench_n4.json
