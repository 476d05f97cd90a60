"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch counts and total time, plus the epoch kernel's per-launch
times.  Usage: python tools/launch_summary.py launches.csv > summary.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iN, iM, iV, iU = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
ep = []
for r in rows[1:]:
    if r[iM] != "gpu__time_duration.sum":
        continue
    v = float(r[iV].replace(",", "")) * scale.get(r[iU], 1e-6 if r[iU] == "nsecond" else 1.0)
    agg[r[iN]][0] += 1
    agg[r[iN]][1] += v
    if "epoch_kernel" in r[iN]:
        ep.append(v)
print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:70]:70s} {n:8d} {t:10.3f}")
print()
print("epoch_kernel per launch (ms): " + " ".join(f"{v:.3f}" for v in ep))
