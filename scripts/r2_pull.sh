#!/usr/bin/env bash
# pull-mode slab + batched consume at N=2; footprint diagnostic; ncu of rank 0's probe kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${1:-2}
tr() { timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for v in "PSG_SLAB_PUSH=0" "PSG_SLAB_PUSH=1" "PSG_SLAB_DIAG=2" "PSG_SLAB_DIAG=10"; do
  env $v bash -c "$(declare -f tr); N=$N; tr scripts/q3_value_mgpu.py --steps 10 --tag '$v'" 2>&1 | grep '^{' | tail -1
done
PSG_TRACE=3 tr scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag trace > gpurun_out/r2_trace_n${N}_pull.txt 2>&1
grep "device" gpurun_out/r2_trace_n${N}_pull.txt | tail -14
cat > /tmp/ncu_r0.sh <<'EOS'
#!/usr/bin/env bash
if [ "$RANK" = "0" ]; then
  exec ncu --set full --import-source on --clock-control none -k regex:psg_jit_scan -s 5 -c 1 -o gpurun_out/r2_probe_slab_n2 python "$@"
else
  exec python "$@"
fi
EOS
chmod +x /tmp/ncu_r0.sh
TMO=600 tr --no-python /tmp/ncu_r0.sh scripts/q3_value_mgpu.py --steps 1 --warmup 1 --tag ncu > gpurun_out/r2_ncu_slab_n2.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r2_ncu_slab_n2.log
