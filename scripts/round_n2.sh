#!/usr/bin/env bash
# 2-GPU box: the N=1 round check (scripts/round_n1.sh) plus N=2 multi-GPU parity.
cd "$(dirname "$0")/.."
bash scripts/round_n1.sh
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29692 scripts/mgpu_check.py --fuzz 60 --sf10 > gpurun_out/mgpu2_final.txt 2>&1
echo "mgpu N=2 rc=$? ok=$(grep -c ' OK' gpurun_out/mgpu2_final.txt) $(grep FAILURES gpurun_out/mgpu2_final.txt)"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29602 bench.py --gpus 2 > gpurun_out/scale_2.json 2> gpurun_out/scale_2.err; echo "bench n2 rc=$?"
