#!/usr/bin/env bash
# 4-GPU: the N>4 default path (SUM all-reduce of the key bitmaps) forced at N=4: parity + value;
# e2e reader threads per rank at N=4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tr() { N=$1; shift; timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
PSG_KB_OR=0 TMO=1500 tr 4 scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu4_parity_kbsum.txt 2>&1
echo "parity4 kbsum rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu4_parity_kbsum.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu4_parity_kbsum.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu4_parity_kbsum.txt | head -5
for v in "PSG_KB_OR=0" "PSG_KB_OR=1"; do env $v bash -c "$(declare -f tr); tr 4 scripts/q3_value_mgpu.py --steps 10 --tag '$v'" 2>&1 | grep -E '^\{|rror' | tail -1; done
for t in 4 6 8; do
  TMO=1200 tr 4 bench.py --gpus 4 --steps 5 --warmup 2 --no-block --budget-gb 0 --io-threads $t 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('T=$t', d['value'], d['e2e']['value'], d['e2e_roofline']['terms'])"
done
