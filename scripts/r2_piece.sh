#!/usr/bin/env bash
# ingest readers sharing batches piece by piece: timeline, e2e, tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PSG_TIMELINE=gpurun_out/tl_n1c timeout 600 python scripts/timeline_run.py 2>&1 | tail -8
timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --budget-gb 0 2>/dev/null | python -c "
import sys, json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('e2e', d['e2e']['value'], 'block', d['e2e_block']['value'], 'ingest_probe', d['e2e_roofline']['terms']['ingest_pipelined_s'], 'value', d['value'], 'parity', d['parity']['match'], d['parity'].get('block_match'))"
for t in 8 16; do timeout 600 python bench.py --steps 5 --warmup 2 --no-block --no-cpu-baseline --budget-gb 0 --io-threads $t 2>/dev/null | python -c "
import sys, json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('T=$t e2e', d['e2e']['value'], 'ingest_probe', d['e2e_roofline']['terms']['ingest_pipelined_s'])"; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_piece.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_gpu_tests_piece.txt
