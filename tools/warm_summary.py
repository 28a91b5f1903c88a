"""Median per-kernel device time from an ncu launch list (gpu__time_duration.sum, ns)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "ID")
i = rows.index(hdr)
d = collections.defaultdict(list)
for r in rows[i + 1:]:
    if len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
        d[r[hdr.index("Kernel Name")].split("(")[0][:48]].append(float(r[hdr.index("Metric Value")]))
for k, v in d.items():
    v.sort()
    print(f"{k:50s} n={len(v):4d} median {v[len(v) // 2] / 1e3:8.2f} us  total {sum(v) / 1e3:9.1f} us")
