"""Mean gpu__time_duration per kernel name from an ncu --csv launch list:
python tools/ncu_kernel_means.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr, rows = rows[0], rows[1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
acc = defaultdict(list)
for r in rows:
    acc[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:60]:60s} n={len(v):4d} mean={sum(v) / len(v) / 1e3:9.2f} us")
