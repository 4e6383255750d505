#!/usr/bin/env bash
# e2e ingest A/B at N=1: file mappings + NT copies vs pread; reader threads
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "PSG_MMAP=1 T=12" "PSG_MMAP=1 T=16" "PSG_MMAP=1 T=8" "PSG_MMAP=0 T=12"; do
  m=$(echo $v | sed 's/.*PSG_MMAP=\([01]\).*/\1/'); t=$(echo $v | sed 's/.*T=//')
  PSG_MMAP=$m timeout 600 python bench.py --steps 5 --warmup 2 --no-block --no-cpu-baseline --budget-gb 0 --io-threads $t 2>/dev/null | python -c "
import sys, json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', 'e2e', d['e2e']['value'], 'ingest_probe', d['e2e_roofline']['terms']['ingest_pipelined_s'], 'value', d['value'])"
done
