#!/usr/bin/env bash
# N-GPU: parity of the current build (mgpu_check incl. random plans and SF10), then an A/B of the
# build insert overlapped with the probe side (PSG_BUILD_OVERLAP) on the staged SF100 Q3 query.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${N:-2}
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29641 \
  scripts/mgpu_check.py --fuzz 60 --sf10 > gpurun_out/mgpu${N}_ov.txt 2>&1; echo "mgpu_check rc=$?"
grep -c " OK" gpurun_out/mgpu${N}_ov.txt; grep -i "fail\|mismatch" gpurun_out/mgpu${N}_ov.txt | head -5
python -c "import sys; sys.path.insert(0,'.'); import bench; bench.ensure_data('/tmp/psg_bench/sf100_n8', 100.0, 8)" > /dev/null 2>&1
for o in ${OVS:-0 1 0 1}; do
  echo "== overlap $o"
  PSG_BUILD_OVERLAP=$o timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29642 scripts/profile_mgpu.py 100 2> gpurun_out/ov_$o.err | grep "^run 3" | python -c "import sys,json; d=json.loads(sys.stdin.read().split(' ',2)[2]); print('device_ms %.3f probe_kernel_ms %.3f' % (d['device_ms'], d['probe_kernel_ms']))"
done
