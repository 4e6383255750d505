#!/usr/bin/env bash
# A/B of engine knobs at one GPU (SF100 HBM-resident query, parity checked):
#   bash scripts/ab_n1.sh "PSG_X=0" "PSG_X=1 PSG_Y=2" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do env $v timeout 300 python scripts/q3_value.py --tag "$v" 2>&1 | tail -1; done
