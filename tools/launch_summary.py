"""Summarise an ncu launch list (gpu__time_duration.sum per launch) of bench.py:
per-kernel totals over the last iteration found (k_fwd ... k_average)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]
ki, vi, idi, gi = h.index('Kernel Name'), h.index('Metric Value'), h.index('ID'), h.index('Grid Size')
data = rows[hdr + 1:]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 21
last = data[-(n + 1):]
tot = 0.0
for r in last:
    t = float(r[vi]) / 1e3
    tot += t
    print(f"{r[idi]:>5} {r[ki][:48]:48s} grid {r[gi]:>14s} {t:10.1f} us")
print(f"total {tot:.1f} us")
