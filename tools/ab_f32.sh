#!/bin/bash
# A/B of describe_f32 build knobs on the GPU box: for each "-DNAME=V ..." set,
# rebuild describe_f32.o and time C2 describe (tools/f32_time.py).
cd "$(dirname "$0")/../paper_2405_08578_b200/csrc"
for flags in "$@"; do
  rm -f build/describe_f32.o
  make -s EXTRA="$flags" >/dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  (cd ../.. && python tools/f32_time.py 64 auto "[$flags]")
done
rm -f build/describe_f32.o && make -s >/dev/null 2>&1
