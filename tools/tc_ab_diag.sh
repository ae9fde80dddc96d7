cd $GRAFT_REPO_ROOT
LIB=paper_2405_08578_b200/libpeakstitch_b200.so
cp $LIB /tmp/keep.so
for v in BASE NOAUG NOEPI NOCOPYNOEPI NOCOPYNOEPINOAUG; do
  cp ab_src/lib_$v.so $LIB
  timeout 300 ncu --kernel-name regex:nn_topk_tc --metrics gpu__time_duration.sum --clock-control none -c 3 --csv python tools/tc_dense.py > gpurun_out/tcab_$v.csv 2> gpurun_out/tcab_$v.err
  echo "== $v"; grep -o '"nn_topk_tc<[01]>[^"]*","[^"]*"' gpurun_out/tcab_$v.csv | head -0
  python - <<PY
import csv
rows=list(csv.reader(l for l in open("gpurun_out/tcab_$v.csv") if l.startswith('"')))
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r))
    print(d["Kernel Name"][:40], d["Grid Size"], d["Metric Value"], d["Metric Unit"])
PY
done
cp /tmp/keep.so $LIB
