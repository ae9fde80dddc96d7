#!/bin/bash
# dense / C5 / C4 matcher timings for each library given: tools/ab_match_all.sh ab_src/lib_X.so ...
cd "$(dirname "$0")/.."
LIB=paper_2405_08578_b200/libpeakstitch_b200.so
cp $LIB /tmp/keep.so
for f in "$@"; do
  cp "$f" $LIB; echo "== $f"
  timeout 300 python tools/tc_dense.py 2>&1 | tail -1 | cut -c1-110
  timeout 300 python tools/c5_time.py x 2>&1 | tail -1
  timeout 300 python tools/profile_c4.py 2>&1 | tail -2
done
cp /tmp/keep.so $LIB
