"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
launches, mean and total microseconds per kernel (first-seen order)."""
import csv
import sys

agg = {}
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            k = d["Kernel Name"].replace("tbt::<unnamed>::", "")[:64]
            agg.setdefault(k, []).append(float(d["Metric Value"]) / 1e3)
for k, v in agg.items():
    print(f"{k:66s} n={len(v):4d} mean={sum(v) / len(v):9.1f}us total={sum(v):10.1f}us")
