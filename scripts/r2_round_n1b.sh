#!/usr/bin/env bash
# N=1 evidence at HEAD: smoke, bench line (identity + block + budget + CPU reference), launch list + ncu of the probe kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2b_smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/r2b_bench_n1.json 2> gpurun_out/r2b_bench_n1.err; echo "bench rc=$?"
cat gpurun_out/r2b_bench_n1.json; tail -3 gpurun_out/r2b_bench_n1.err
timeout 900 bash scripts/profile_n1.sh
