#!/usr/bin/env bash
# N=1 evidence for profiles/: launch list of one staged SF100 Q3 query (second of two) and an
# ncu --set full capture of its dominant kernel (the largest psg_jit_scan launch).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/profile_q3.py --warmup 1 --steps 1 > gpurun_out/pq3.log 2>&1 || { echo "profile_q3 failed"; tail gpurun_out/pq3.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv \
  python scripts/profile_q3.py --warmup 1 --steps 1 > /dev/null 2>&1
IDX=$(python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/launches_n1.csv")) if r]
hdr = next(r for r in rows if r[0] == "ID")
ks = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "ID"]
jit = [k for k in ks if "psg_jit_scan" in k["Kernel Name"]]
half = jit[len(jit) // 2:]  # the second query's launches
best = max(range(len(half)), key=lambda i: float(half[i]["Metric Value"].replace(",", "")))
print(len(jit) // 2 + best)
PY
)
echo "probe kernel = psg_jit_scan launch $IDX"
ncu --set full --import-source on --clock-control none -k regex:psg_jit_scan -s $IDX -c 1 -o gpurun_out/probe_full \
  python scripts/profile_q3.py --warmup 1 --steps 1 > gpurun_out/ncu_probe.log 2>&1
tail -2 gpurun_out/ncu_probe.log
python scripts/launches.py gpurun_out/launches_n1.csv $(( $(grep -c gpu__time_duration gpurun_out/launches_n1.csv) / 2 )) | tail -25
