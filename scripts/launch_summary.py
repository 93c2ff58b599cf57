"""Per-kernel launch counts and mean ncu durations from a launch-list CSV
(ncu --metrics gpu__time_duration.sum --csv): launch_summary.py FILE."""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
d = collections.defaultdict(list)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1e3 if r[ui] == "ms" else 1)
    m = re.search(r"(\w+_kernel)\b", r[ki])
    d[m.group(1) if m else r[ki][:40]].append(v)
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:44s} n={len(v):4d} mean={sum(v) / len(v):8.1f} us  total={sum(v) / 1e3:7.2f} ms")
