#!/usr/bin/env bash
# Runs bench.py at N = 1 .. $1 GPUs back to back (one JSON line per N in gpurun_out/scale_N.json).
MAXN=${1:-4}
python bench.py > gpurun_out/scale_1.json 2> gpurun_out/scale_1.err
for N in 2 4 8; do
  [ "$N" -le "$MAXN" ] || break
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + N)) bench.py --gpus $N > gpurun_out/scale_$N.json 2> gpurun_out/scale_$N.err
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_1.json 2> gpurun_out/ref_1.err
