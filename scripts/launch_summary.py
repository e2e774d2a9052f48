"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (per-kernel share)."""
import collections
import csv
import sys

path = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in data:
    name = r[ki].split("(")[0].replace("void ", "")[:48]
    tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':48s} {'launches':>8s} {'us/step':>10s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:48s} {cnt[k]:8d} {v / steps:10.1f} {100 * v / T:5.1f}%")
print(f"{'total':48s} {sum(cnt.values()):8d} {T / steps:10.1f}")
