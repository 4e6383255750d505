#!/usr/bin/env bash
# 4-GPU box evidence at HEAD: parity N=4 and N=2, bench lines N=2 and N=4 (identity headline +
# block codec + budget + modes), phase traces, e2e timelines at N=4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tr() { N=$1; shift; timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for N in 4 2; do
  TMO=1500 tr $N scripts/mgpu_check.py --fuzz 20 --sf10 > gpurun_out/rf_mgpu${N}_parity.txt 2>&1
  echo "parity$N rc=$? ok=$(grep -c ' OK' gpurun_out/rf_mgpu${N}_parity.txt) bad=$(grep -c 'BAD' gpurun_out/rf_mgpu${N}_parity.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/rf_mgpu${N}_parity.txt | head -5
  TMO=1500 tr $N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/rf_bench_n${N}.json 2> gpurun_out/rf_bench_n${N}.err; echo "bench$N rc=$?"
  tail -1 gpurun_out/rf_bench_n${N}.json | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['e2e']['value'], (d.get('e2e_block') or {}).get('value'), d['roofline']['frac'], d['parity'], d.get('e2e_modes'))"
  PSG_TRACE=3 tr $N scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace > gpurun_out/rf_trace_n${N}.txt 2>&1
done
PSG_TIMELINE=gpurun_out/tl_n4 tr 4 scripts/timeline_run.py 2>&1 | tail -8
