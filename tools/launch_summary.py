"""Summarise an ncu --metrics gpu__time_duration.sum CSV into per-kernel shares."""
import collections
import csv
import re
import sys

path = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0  # e.g. number of horizons captured
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in data:
    name = re.sub(r"\(.*", "", r[ki]).replace("enks::<unnamed>::", "")[:70]
    tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
    cnt[name] += 1
T = sum(tot.values())
print(f"{'us/unit':>12} {'share':>6} {'launches':>8}  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / div:12.1f} {100 * v / T:5.1f}% {cnt[k] / div:8.1f}  {k}")
print(f"{T / div:12.1f} total us/unit")
