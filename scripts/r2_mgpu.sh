#!/usr/bin/env bash
# N-GPU box (N=2 or 4): quick N=1 check of the current build, multi-GPU parity (random plans, SF10,
# duplicate-key plans, join microbenchmark vs the reference per node), the A/B of the N>1
# aggregation-table variants at SF100, the N-GPU bench line and the join microbenchmark at N.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${1:-2}
nvidia-smi topo -m 2>&1 | head -6
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
CUDA_VISIBLE_DEVICES=0 timeout 300 python scripts/q3_value.py --tag n1 2>&1 | tail -1
TMO=1500 tr scripts/mgpu_check.py --fuzz 40 --sf10 > gpurun_out/r2_mgpu${N}_parity.txt 2>&1
echo "parity rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu${N}_parity.txt) bad=$(grep -c 'BAD' gpurun_out/r2_mgpu${N}_parity.txt)"; grep -E "BAD|FAIL|Error" gpurun_out/r2_mgpu${N}_parity.txt | head -5
for v in "PSG_RANK_TABLE=1" "PSG_RANK_TABLE=0" "PSG_RANK_TABLE=0 PSG_KBITS=2" "PSG_RANK_TABLE=1 PSG_PACK=0" "PSG_TMA_MAT=1"; do
  echo "== $v"; env $v bash -c "$(declare -f tr); N=$N; tr scripts/q3_value_mgpu.py --tag '$v'" 2>&1 | grep '^{' | tail -1
done
TMO=1200 tr bench.py --gpus $N --steps 10 --warmup 3 --no-block > gpurun_out/r2_bench_n${N}.json 2> gpurun_out/r2_bench_n${N}.err; echo "bench rc=$?"
tail -c 3500 gpurun_out/r2_bench_n${N}.json
tr scripts/join_bench.py > gpurun_out/r2_join_n${N}.json 2> gpurun_out/r2_join_n${N}.err; echo "join rc=$?"
cat gpurun_out/r2_join_n${N}.json; tail -3 gpurun_out/r2_join_n${N}.err
