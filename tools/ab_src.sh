#!/bin/bash
# A/B of describe_f32.cu source variants on the GPU box: for each file given
# (e.g. ab_src/*.cu), build it in place of csrc/describe_f32.cu and time C2
# describe (tools/f32_time.py); the working copy is restored afterwards.
REPO="$(cd "$(dirname "$0")/.." && pwd)"
CS="$REPO/paper_2405_08578_b200/csrc"
cp "$CS/describe_f32.cu" /tmp/describe_f32.cu.keep
for f in "$@"; do
  for rep in 1 2; do
    cp "$REPO/$f" "$CS/describe_f32.cu"
    rm -f "$CS/build/describe_f32.o"
    make -s -C "$CS" >/dev/null 2>&1 || { echo "build failed: $f"; continue; }
    (cd "$REPO" && python tools/f32_time.py 64 auto "[$f #$rep]")
  done
done
cp /tmp/describe_f32.cu.keep "$CS/describe_f32.cu"
rm -f "$CS/build/describe_f32.o" && make -s -C "$CS" >/dev/null 2>&1
