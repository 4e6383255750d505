#!/usr/bin/env bash
# N-GPU parity (mgpu_check incl. staged runs, random plans, SF10) + A/B of the chunked probe pipeline.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${N:-2}
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29681 \
  scripts/mgpu_check.py --fuzz 60 --sf10 > gpurun_out/mgpu${N}_chunks.txt 2>&1; echo "mgpu_check rc=$?"
grep -c " OK" gpurun_out/mgpu${N}_chunks.txt; grep -i "BAD\|FAILURES\|error" gpurun_out/mgpu${N}_chunks.txt | head -8
ENVVAR=PSG_PROBE_CHUNKS VALS="${VALS:-1 4 2 8 1 4}" N=$N bash scripts/ab_env_mgpu.sh
