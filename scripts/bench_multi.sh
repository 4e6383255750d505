#!/usr/bin/env bash
# bench.py at N = 2 and 4 for the identity and block codecs (gpurun_out/scale_N.json, blk_N.json).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + N)) bench.py --gpus $N > gpurun_out/scale_$N.json 2> gpurun_out/scale_$N.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29700 + N)) bench.py --gpus $N --codec block > gpurun_out/blk_$N.json 2> gpurun_out/blk_$N.err
done
for f in gpurun_out/scale_[24].json gpurun_out/blk_[24].json; do
  echo "$f: $(tail -1 $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d.get('value'), d.get('e2e',{}).get('value'), d.get('roofline',{}).get('frac'), d['config'].get('batch_mb'), d.get('clocks'))" 2>&1)"
done
