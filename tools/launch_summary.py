"""Summarise an ncu --csv launch list (gpu__time_duration.sum): total time,
count and share per kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
acc, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0][:70]
        acc[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
tot = sum(acc.values())
print(f"total {tot / 1e3:.1f} us over {sum(cnt.values())} launches")
for k, v in sorted(acc.items(), key=lambda x: -x[1])[:40]:
    print(f"{v / 1e3:10.1f} us {100 * v / tot:5.1f} % {cnt[k]:5d}x  {k}")
