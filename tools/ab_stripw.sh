LIB=paper_2405_08578_b200/libpeakstitch_b200.so
cp $LIB /tmp/keep.so
for f in ab_src/lib_NS*.so; do cp $f $LIB; echo "== $f"; python tools/det_speed.py 2>&1 | grep "C4"; done
cp /tmp/keep.so $LIB
