#!/usr/bin/env bash
# distributed-join microbenchmark (the reference's four run_join schedules) at N = 1, 2, 4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 900 python scripts/join_bench.py > gpurun_out/r2_join_n1.json 2> gpurun_out/r2_join_n1.err; echo "n1 rc=$?"; cat gpurun_out/r2_join_n1.json
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + N)) scripts/join_bench.py > gpurun_out/r2_join_n$N.json 2> gpurun_out/r2_join_n$N.err; echo "n$N rc=$?"; cat gpurun_out/r2_join_n$N.json
done
