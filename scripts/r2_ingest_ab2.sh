#!/usr/bin/env bash
# e2e ingest A/B at N=1: batch size x reader threads (file mappings + NT copies)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "64 8" "64 12" "32 12" "256 12" "128 10"; do
  set -- $v
  timeout 600 python bench.py --steps 5 --warmup 2 --no-block --no-cpu-baseline --budget-gb 0 --batch-mb $1 --io-threads $2 2>/dev/null | python -c "
import sys, json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('batch $1 T=$2', 'e2e', d['e2e']['value'], 'ingest_probe', d['e2e_roofline']['terms']['ingest_pipelined_s'], 'value', d['value'])"
done
