"""profiles/traffic.json from an ncu launch list (dram bytes of the describe
kernel per launch) and an `ncu --set full --page raw --csv` export of one
describe launch.  usage: make_traffic.py LAUNCHES.csv RAW.csv RAW_NAME"""
import csv
import json
import sys

launches, raw, raw_name = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(l for l in open(launches) if l.startswith('"')))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = {}
for r in rows[1:]:
    if "describe_pair_kernel" in r[ki] and r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v = float(r[vi].replace(",", ""))
        unit = r[h.index("Metric Unit")]
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        per[r[ii]] = per.get(r[ii], 0.0) + v
dram = sum(per.values()) / len(per)
R = list(csv.reader(open(raw)))
hdr, val = R[0], R[2]
get = lambda k: float(val[hdr.index(k)].replace(",", ""))  # noqa: E731
out = {"describe_kernel": {
    "images": 64, "dram_bytes_per_launch": int(dram),
    "source": f"{launches.split('/')[-1]}: ncu dram__bytes_read.sum + dram__bytes_write.sum of describe_pair_kernel, "
              "mean over launches",
    "ncu_full": {"issue_active_frac": round(get("smsp__issue_active.avg.pct_of_peak_sustained_active") / 100, 4),
                 "fp64_pipe_frac": round(get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") / 100, 4),
                 "warps_active_frac": round(get("sm__warps_active.avg.pct_of_peak_sustained_active") / 100, 4),
                 "warp_instructions": int(get("smsp__inst_executed.sum")),
                 "source": f"profiles/{raw_name} (ncu --set full, one launch)"}}}
print(json.dumps(out, indent=1))
