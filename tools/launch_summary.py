"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launch count, total ms, share.  usage: launch_summary.py file.csv [top]"""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[1:]:
    name = r[ki].split("(")[0].split("::")[-1]
    v = float(r[vi].replace(",", ""))
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{len(rows) - 1} launches, {T / 1e6:.2f} ms total (serialised, cold-cache)")
for k, v in sorted(tot.items(), key=lambda t: -t[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"  {k:28s} {cnt[k]:6d} {v / 1e6:9.3f} ms {100 * v / T:5.1f}%")
