#!/usr/bin/env bash
# 4-GPU box at HEAD: parity N=4, values N=2/N=4 (+NCCL path), traces, bench lines N=2 and N=4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tr() { N=$1; shift; timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
TMO=1500 tr 4 scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu4_parity_b.txt 2>&1
echo "parity4 rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu4_parity_b.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu4_parity_b.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu4_parity_b.txt | head -5
tr 4 scripts/q3_value_mgpu.py --steps 10 --tag n4 2>&1 | grep '^{' | tail -1
PSG_SLAB=0 tr 4 scripts/q3_value_mgpu.py --steps 10 --tag n4_noslab 2>&1 | grep '^{' | tail -1
PSG_TRACE=3 tr 4 scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace > gpurun_out/r2_trace_n4b.txt 2>&1
grep "device" gpurun_out/r2_trace_n4b.txt | tail -15
TMO=1200 tr 4 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r2b_bench_n4.json 2> gpurun_out/r2b_bench_n4.err; echo "bench4 rc=$?"
TMO=1200 tr 2 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2b_bench_n2.json 2> gpurun_out/r2b_bench_n2.err; echo "bench2 rc=$?"
for f in gpurun_out/r2b_bench_n4.json gpurun_out/r2b_bench_n2.json; do tail -1 $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['e2e']['value'], (d.get('e2e_block') or {}).get('value'), d['roofline']['frac'], d['parity']['match'], d['shuffle'])"; done
