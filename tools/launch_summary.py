"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): count, total ms and
share of GPU time per kernel.   python tools/launch_summary.py launches.csv [header line]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    v = v / 1e6 if r[ui] in ("nsecond", "ns") else v / 1e3 if r[ui] in ("usecond", "us") else v
    tot[r[ki]] += v
    cnt[r[ki]] += 1
all_ms = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print("count  total_ms  share  kernel")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{cnt[k]:5d} {tot[k]:9.3f} {100 * tot[k] / all_ms:5.1f}%  {k[:80]}")
