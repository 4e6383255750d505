#!/usr/bin/env bash
# A/B of the fused scan kernels' CTAs-per-SM (register cap) on the staged SF100 Q3 query (N=1).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); import bench; bench.ensure_data('/tmp/psg_bench/sf100_n8', 100.0, 8)" > /dev/null 2>&1
for m in ${MINBS:-8 7 6 5}; do
  echo "== minb $m"
  PSG_JIT_MINB=$m PSG_TRACE=1 python scripts/profile_q3.py --scale 100 --warmup 2 --steps 3 2> gpurun_out/minb_$m.err | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('device_ms %.3f probe_kernel_ms %.3f' % (d['device_ms'], d['probe_kernel_ms']))"
  grep "jit kernel" gpurun_out/minb_$m.err | sort | uniq
done
