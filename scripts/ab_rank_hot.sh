#!/usr/bin/env bash
# A/B of the rank-table hot-slot writer (PSG_RANK_HOT_SEQ) at SF100 N=1: parity on the golden
# cases, query device time, and the k_rank_* kernel times from an ncu launch list per setting.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PSG_RANK_HOT_SEQ=1 python scripts/golden_check.py 2>&1 | grep -E "BAD|Traceback" | tail -2
ENVVAR=PSG_RANK_HOT_SEQ VALS="0 1 0 1 0 1" bash scripts/ab_env.sh
for v in 0 1; do
  PSG_RANK_HOT_SEQ=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:k_rank --csv --log-file gpurun_out/rank_hot$v.csv \
    python scripts/profile_q3.py --warmup 1 --steps 1 > /dev/null 2>&1
  echo "HOT_SEQ=$v:"; grep -o '"k_rank[^"]*\|"gpu__time_duration.sum","[^"]*","[^"]*"\|"dram__bytes_[a-z]*.sum","[^"]*","[^"]*"' gpurun_out/rank_hot$v.csv | tail -8 | tr '\n' ' '; echo
done
