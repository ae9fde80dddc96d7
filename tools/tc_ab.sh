#!/bin/bash
# nn_topk_tc launch times (ncu launch list, dense 103,968^2 match) for each
# library given: tools/tc_ab.sh ab_src/lib_X.so ...
cd "$(dirname "$0")/.."
LIB=paper_2405_08578_b200/libpeakstitch_b200.so
cp $LIB /tmp/keep.so
for f in "$@"; do
  cp "$f" $LIB
  timeout 300 ncu --kernel-name regex:nn_topk_tc --metrics gpu__time_duration.sum --clock-control none -c 3 --csv \
    python tools/tc_dense.py > /tmp/tcab.csv 2> /tmp/tcab.err
  echo "== $f"
  python - <<PY
import csv
rows=list(csv.reader(l for l in open("/tmp/tcab.csv") if l.startswith('"')))
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r))
    print(d["Kernel Name"][:22], d["Grid Size"], d["Metric Value"], d["Metric Unit"])
PY
  timeout 300 python tools/tc_dense.py | tail -1
done
cp /tmp/keep.so $LIB
