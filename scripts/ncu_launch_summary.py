"""Per-kernel totals of an ncu launch list (`--metrics gpu__time_duration.sum
--csv --log-file X.csv`):  python scripts/ncu_launch_summary.py X.csv [steps]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot, cnt = collections.OrderedDict(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("unnamed>::", "")
    name = re.sub(r"fc2t2::\(anonymous namespace\)::", "", name)
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot[name] = tot.get(name, 0.0) + v
    cnt[name] += 1
allt = sum(tot.values())
print(f"serialised total {allt / steps:.1f} us per step ({sum(cnt.values()) / steps:.0f} launches)")
print(f"{'us/step':>9} {'launches':>8} {'share':>6}  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / steps:9.1f} {cnt[k] / steps:8.1f} {100 * v / allt:5.1f}%  {k}")
