#!/usr/bin/env bash
# 1-GPU box: finer N=1 phase trace, and the zero-copy / NT-copy ingest probe on the SF100 files.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PSG_TRACE=3 timeout 300 python scripts/q3_value.py --steps 1 --warmup 1 --tag trace1 > gpurun_out/r2_trace_n1b.txt 2>&1
df -T /tmp /dev/shm > gpurun_out/r2_ingest_probe2.txt; nproc >> gpurun_out/r2_ingest_probe2.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/r2_ingest_probe2.txt
free -g >> gpurun_out/r2_ingest_probe2.txt
cat /tmp/psg_bench/sf100_n8/dev*/*.psto > /dev/null
timeout 600 ./scripts/ingest_probe2 /tmp/psg_bench/sf100_n8/dev*/lineitem*.psto /tmp/psg_bench/sf100_n8/dev*/orders*.psto >> gpurun_out/r2_ingest_probe2.txt 2>&1
echo "probe rc=$?"; cat gpurun_out/r2_ingest_probe2.txt
