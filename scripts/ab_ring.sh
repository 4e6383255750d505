#!/usr/bin/env bash
# A/B of the HBM ring depth (PSG_RING_SLOTS) and batch size on the e2e at N=1 (CODEC=block|identity).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for codec in ${CODECS:-block}; do
python bench.py --codec $codec --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
for cfg in ${CFGS:-"8 64" "16 64" "24 64" "16 128" "8 64"}; do
  set -- $cfg
  echo "== $codec slots $1 batch_mb $2: $(PSG_RING_SLOTS=$1 python bench.py --codec $codec --batch-mb $2 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])")"
done
done
