#!/usr/bin/env bash
# torchrun --no-python scripts/ncu_rank0.sh <script.py> [args]: rank 0 runs under ncu with a
# single-pass DRAM metric set on ONE launch of the fused probe kernel (-s/-c from NCU_SKIP, default
# 5: the probe of the second query of q3_value_mgpu.py), so NCCL and the peers proceed as in a
# normal run; the other ranks run plainly. Output: gpurun_out/ncu_rank0_n${WORLD_SIZE}.csv
if [ "$RANK" = "0" ]; then
  exec ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:psg_jit_scan -s ${NCU_SKIP:-5} -c 1 --csv --log-file gpurun_out/ncu_rank0_n${WORLD_SIZE}.csv python "$@"
else
  exec python "$@"
fi
