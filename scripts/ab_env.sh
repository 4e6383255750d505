#!/usr/bin/env bash
# A/B of an engine env knob on the staged SF100 Q3 query at N=1: ENVVAR=name VALS="0 1 0 1".
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); import bench; bench.ensure_data('/tmp/psg_bench/sf100_n8', 100.0, 8)" > /dev/null 2>&1
for v in ${VALS:-0 1 0 1}; do
  echo "== $ENVVAR=$v: $(env $ENVVAR=$v python scripts/profile_q3.py --scale 100 --warmup 2 --steps 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('device_ms %.3f probe_kernel_ms %.3f' % (d['device_ms'], d['probe_kernel_ms']))")"
done
