#!/usr/bin/env bash
# N=2/N=4 box: multi-GPU parity (60 random plans + SF10 vs the reference per node) and the A/B of
# the N>1 aggregation table variants at SF100.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${1:-2}
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
timeout 1500 tr scripts/mgpu_check.py --fuzz 60 --sf10 > gpurun_out/r2_mgpu${N}_parity.txt 2>&1
echo "parity rc=$? ok=$(grep -c ' OK' gpurun_out/r2_mgpu${N}_parity.txt) $(grep -E 'FAIL|BAD' gpurun_out/r2_mgpu${N}_parity.txt | head -3)"
run() { echo "== $*"; env "$@" timeout 600 bash -c "$(declare -f tr); N=$N; tr scripts/q3_value_mgpu.py --tag '$*'" 2>&1 | grep '^{' | tail -1; }
run PSG_RANK_TABLE=1
run PSG_RANK_TABLE=0
run PSG_RANK_TABLE=0 PSG_KBITS=2
run PSG_RANK_TABLE=1 PSG_PACK=0
run PSG_RANK_TABLE=1
