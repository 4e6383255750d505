#!/usr/bin/env bash
# A/B of the GPU inflate kernel: the working tree's libpsg.so vs ab/libpsg_old.so (built from the
# previous commit), on the same box: stage (one launch over every SF10 lineitem/orders chunk) and
# end-to-end block-codec query times, then the k_inflate launch time under ncu (cold, serialised).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
[ -n "$SKIP_TESTS" ] || python -m pytest tests/test_gpu_codec.py -x -q 2>&1 | tail -3
rm -rf /tmp/oldrepo && cp -r . /tmp/oldrepo && cp ab/libpsg_old.so /tmp/oldrepo/paper_2512_02862_b200/libpsg.so
for v in new old; do
  R=.; [ $v = old ] && R=/tmp/oldrepo
  python $R/scripts/inflate_probe.py --scale ${SCALE:-10} --steps 3 > gpurun_out/ip_$v.log 2>&1
done
for v in new old; do
  R=.; [ $v = old ] && R=/tmp/oldrepo
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_inflate -c 6 --csv \
    python $R/scripts/inflate_probe.py --scale ${SCALE:-10} --steps 1 > gpurun_out/ip_${v}_ncu.csv 2>&1
done
for v in new old; do echo "== $v"; cat gpurun_out/ip_$v.log; grep gpu__time_duration gpurun_out/ip_${v}_ncu.csv | cut -d, -f8,15; done
