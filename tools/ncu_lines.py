"""Summarise an `ncu --page source --csv --print-source cuda,sass` export:
instructions and stall samples per CUDA source line, and the SASS opcode mix."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = collections.OrderedDict()
ops = collections.Counter()
ie = ws = None
fname = ""
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        ie = r.index("Instructions Executed")
        ws = r.index("Warp Stall Sampling (All Samples)")
        continue
    try:
        if r[0] != "":
            cur = (fname, int(r[0]), r[1].strip()[:100])
            agg[cur] = [float(r[ie] or 0), float(r[ws] or 0)]
        else:
            m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", r[3])
            if m:
                ops[m.group(1)] += float(r[ie] or 0)
    except (ValueError, IndexError):
        continue  # multi-line source text
tot = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values()) or 1
print("total warp instructions", tot)
for (f, l, s), (v, w) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * v / tot:5.1f}% inst {100 * w / ts:5.1f}% stall  {f}:{l}: {s}")
print()
tot_ops = sum(ops.values())
for o, v in ops.most_common(30):
    print(f"{o:14s} {100 * v / tot_ops:5.1f}%")
