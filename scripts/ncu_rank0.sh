#!/usr/bin/env bash
# torchrun --no-python scripts/ncu_rank0.sh <script.py> [args]: rank 0 runs under ncu with a
# single-pass metric set (no kernel replay, so NCCL and peer-memory stores behave as in a normal
# run); the other ranks run plainly. Output: gpurun_out/ncu_rank0_n${WORLD_SIZE}.csv
if [ "$RANK" = "0" ]; then
  exec ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"psg_jit_scan|k_slab_consume|k_bucket_emit" --csv --log-file gpurun_out/ncu_rank0_n${WORLD_SIZE}.csv python "$@"
else
  exec python "$@"
fi
