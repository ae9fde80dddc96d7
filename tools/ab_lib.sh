#!/bin/bash
# A/B of whole built libraries on the GPU box: for each .so given, install it
# in place of the package's library and run the command in $AB_CMD (default:
# C5 pairs through bench.py's function); the original library is restored.
REPO="$(cd "$(dirname "$0")/.." && pwd)"
LIB="$REPO/paper_2405_08578_b200/libpeakstitch_b200.so"
cp "$LIB" /tmp/lib.keep
CMD="${AB_CMD:-python tools/c5_time.py}"
for f in "$@"; do
  for rep in 1 2; do
    cp "$REPO/$f" "$LIB"
    (cd "$REPO" && $CMD "[$f #$rep]")
  done
done
cp /tmp/lib.keep "$LIB"
