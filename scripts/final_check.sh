#!/usr/bin/env bash
# Round-end checks on a 4-GPU box: smoke, multi-GPU parity at N=2 and N=4 (streaming + staged,
# random plans, SF10), then the bench refresh (identity + block codec at N=1/2/4, reference arm).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for N in 2 4; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29690 + N)) scripts/mgpu_check.py --fuzz 60 --sf10 > gpurun_out/mgpu${N}_final.txt 2>&1
  echo "mgpu N=$N rc=$? ok=$(grep -c ' OK' gpurun_out/mgpu${N}_final.txt) $(grep FAILURES gpurun_out/mgpu${N}_final.txt)"
done
bash scripts/scale_bench_all.sh 4
