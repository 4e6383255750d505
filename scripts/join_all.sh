#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + N)) scripts/join_bench.py --repeat 2 > gpurun_out/r2_join_n$N.json 2> gpurun_out/r2_join_n$N.err; echo "n$N rc=$?"; cat gpurun_out/r2_join_n$N.json
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 --no-python scripts/ncu_rank0.sh scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag ncu > gpurun_out/r2_ncu_rank0_n2.log 2>&1; echo "ncu rc=$?"; cat gpurun_out/ncu_rank0_n2.csv 2>/dev/null | tail -5
