#!/usr/bin/env bash
# N-GPU A/B of an engine env knob on the staged SF100 Q3 query: ENVVAR=name VALS="0 1 0 1" N=2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${N:-2}
python -c "import sys; sys.path.insert(0,'.'); import bench; bench.ensure_data('/tmp/psg_bench/sf100_n8', 100.0, 8)" > /dev/null 2>&1
for v in ${VALS:-0 1 0 1}; do
  echo "== $ENVVAR=$v: $(env $ENVVAR=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29651 scripts/profile_mgpu.py 100 2>/dev/null | grep "^run 3" | python -c "import sys,json; d=json.loads(sys.stdin.read().split(' ',2)[2]); print('device_ms %.3f probe_kernel_ms %.3f' % (d['device_ms'], d['probe_kernel_ms']))")"
done
