#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "PSG_TMA_NS=4" "PSG_TMA_NS=6" "PSG_TMA_NS=8" "PSG_TMA_NS=3" "PSG_TMA_NG=3 PSG_TMA_CTAS=1" "PSG_TMA_CTAS=3" "PSG_TMA_NG=1 PSG_TMA_CTAS=4" "PSG_TMA_R=8"; do
  env $v timeout 300 python scripts/q3_value.py --tag "$v" 2>&1 | tail -1; done
