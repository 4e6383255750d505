#!/usr/bin/env bash
# ncu --set full of the rank-table build kernels (k_rank_hot, k_rank_build) of one SF100 N=1 query.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_rank -c 2 -o gpurun_out/rank_full \
  python scripts/profile_q3.py --warmup 0 --steps 1 > gpurun_out/ncu_rank.log 2>&1
tail -2 gpurun_out/ncu_rank.log
