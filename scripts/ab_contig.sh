#!/usr/bin/env bash
# A/B of contiguous tile ranges per CTA for the warp-staged compaction (PSG_CONTIG_TILES) at SF100
# N=1: parity, query device time, per-kernel times from an ncu launch list per setting.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PSG_CONTIG_TILES=1 python scripts/golden_check.py 2>&1 | grep -E "BAD|Traceback" | tail -2
PSG_CONTIG_TILES=1 timeout 900 python -m pytest tests/test_gpu_q3.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -1
ENVVAR=PSG_CONTIG_TILES VALS="0 1 0 1 0 1" bash scripts/ab_env.sh
for v in 0 1; do
  PSG_CONTIG_TILES=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/contig$v.csv python scripts/profile_q3.py --warmup 1 --steps 1 > /dev/null 2>&1
  echo "CONTIG=$v:"; python scripts/launches.py gpurun_out/contig$v.csv $(( $(grep -c gpu__time_duration gpurun_out/contig$v.csv) / 2 )) | grep -E "jit_scan|rank|total"
done
