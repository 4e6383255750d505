#!/usr/bin/env bash
# Round-end refresh: bench.py at N = 1, 2, 4 for the identity (headline) and block codecs, plus the
# reference arm. One JSON line per run in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/scale_bench.sh ${1:-4}
for N in 1 2 4; do
  [ "$N" -le "${1:-4}" ] || break
  if [ $N = 1 ]; then
    python bench.py --codec block > gpurun_out/blk_$N.json 2> gpurun_out/blk_$N.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29700 + N)) bench.py --gpus $N --codec block > gpurun_out/blk_$N.json 2> gpurun_out/blk_$N.err
  fi
done
for f in gpurun_out/scale_*.json gpurun_out/blk_*.json gpurun_out/ref_1.json; do
  echo "$f: $(tail -1 $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d.get('value'), d.get('e2e',{}).get('value'), d.get('roofline',{}).get('frac'), d.get('clocks'))" 2>&1)"
done
