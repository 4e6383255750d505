#!/usr/bin/env bash
# chunked outbox: fake (1 GPU) timing + ncu, then N=2 value/parity
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PSG_SLAB_FAKE=1 timeout 300 python scripts/q3_value.py --tag fake 2>&1 | tail -1
PSG_SLAB_FAKE=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:psg_jit_scan -s 5 -c 1 -o gpurun_out/r2_probe_fake2 \
  python scripts/q3_value.py --steps 1 --warmup 1 --tag ncu > gpurun_out/r2_ncu_fake2.log 2>&1; echo "ncu rc=$?"
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
tr scripts/q3_value_mgpu.py --steps 10 --tag n2 2>&1 | grep -E '^\{|rror' | tail -2
PSG_TRACE=3 tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace > gpurun_out/r2_trace_n2_chunk.txt 2>&1
grep "device\|jit kernel" gpurun_out/r2_trace_n2_chunk.txt | tail -16
TMO=1500 tr scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu2_parity_chunk.txt 2>&1
echo "parity rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu2_parity_chunk.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu2_parity_chunk.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu2_parity_chunk.txt | head -5
