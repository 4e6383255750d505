#!/usr/bin/env bash
# PSG_OWN_TABLE A/B at N=4 and per-node parity at N=4 / N=2 (periodic ownership masks in k_or_own)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/ab_mgpu_quick.sh 4 "PSG_OWN_TABLE=1" "PSG_OWN_TABLE=0" "PSG_OWN_TABLE=1" "PSG_OWN_TABLE=0"
tr() { N=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for N in 4 2; do
  tr $N scripts/mgpu_check.py --fuzz 5 > gpurun_out/ot_parity$N.txt 2>&1
  echo "parity$N rc=$? ok=$(grep -c ' OK' gpurun_out/ot_parity$N.txt) bad=$(grep -c BAD gpurun_out/ot_parity$N.txt)"
done
