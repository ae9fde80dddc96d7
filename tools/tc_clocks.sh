#!/bin/bash
# per-tile cycle breakdown of the dense top-4 pass (diagnostic -DPS_TC_DIAG_CLOCKS libraries): tools/tc_clocks.sh ab_src/lib_X.so ...
cd "$(dirname "$0")/.."
LIB=paper_2405_08578_b200/libpeakstitch_b200.so
cp $LIB /tmp/keep.so
for f in "$@"; do cp "$f" $LIB; echo "== $f"; timeout 300 python tools/tc_dense.py 2>&1 | grep -E "^\[issuer|^\[epilogue|^n=" | sort | uniq -c | sort -rn | head -8; done
cp /tmp/keep.so $LIB
