cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_n1.json
python bench.py --codec block > gpurun_out/blk_1.json 2> gpurun_out/blk_1.err; echo "blk rc=$?"
python bench.py --impl reference > gpurun_out/ref_1.json 2> gpurun_out/ref_1.err; echo "ref rc=$?"; tail -1 gpurun_out/ref_1.json
bash scripts/profile_n1.sh
