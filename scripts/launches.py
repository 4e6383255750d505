"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (last step's kernels)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n_last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr, out = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((int(d["ID"]), d["Kernel Name"][:58], float(d["Metric Value"].replace(",", "")) / 1e3))
step = out[-n_last:] if n_last else out
tot = sum(x[2] for x in step)
for o in step:
    print("%4d %-58s %10.1f us %5.1f%%" % (o[0], o[1], o[2], 100 * o[2] / tot))
print("kernels %d, total %.1f us" % (len(step), tot))
