#!/bin/bash
# A/B timing of library variants in variants/*.so on the C2 describe step
for f in variants/*.so; do
  cp "$f" paper_2405_08578_b200/libpeakstitch_b200.so
  echo -n "$f: "
  python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-match --no-stitch 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels']['describe_kernel']['ms'])"
done
