#!/usr/bin/env bash
# Execution timelines (PSG_TIMELINE) of the warm e2e SF100 query at N=1 and N=2, identity and
# block codec; summaries into gpurun_out/timelines.txt, traces into gpurun_out/tl/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/tl
: > gpurun_out/timelines.txt
for codec in identity block; do
  sfx=$([ $codec = identity ] && echo "" || echo "_block")
  echo "== n1$sfx" >> gpurun_out/timelines.txt
  PSG_TIMELINE=gpurun_out/tl/n1$sfx python scripts/timeline_run.py --codec $codec >> gpurun_out/timelines.txt 2>&1
  echo "== n2$sfx" >> gpurun_out/timelines.txt
  PSG_TIMELINE=gpurun_out/tl/n2$sfx timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29671 scripts/timeline_run.py --codec $codec >> gpurun_out/timelines.txt 2>&1
done
grep -v "^\[\|NCCL\|OMP\|\*\*\*" gpurun_out/timelines.txt
