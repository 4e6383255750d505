#!/usr/bin/env bash
# N-GPU A/B of the fused scan kernels' CTAs-per-SM (staged SF100 Q3, PSG_TRACE off).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${N:-2}
python -c "import sys; sys.path.insert(0,'.'); import bench; bench.ensure_data('/tmp/psg_bench/sf100_n8', 100.0, 8)" > /dev/null 2>&1
for m in ${MINBS:-8 6 8 6}; do
  echo "== minb $m"
  PSG_JIT_MINB=$m timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29631 scripts/profile_mgpu.py 100 2> gpurun_out/minbm_$m.err | grep "^run 3" | python -c "import sys,json; d=json.loads(sys.stdin.read().split(' ',2)[2]); print('device_ms %.3f probe_kernel_ms %.3f' % (d['device_ms'], d['probe_kernel_ms']))"
done
