#!/bin/bash
# A/B timing of library variants in abvar/*.so on the C2 describe step
# (each variant ROUNDS times, interleaved); restores the in-tree build after.
cp paper_2405_08578_b200/libpeakstitch_b200.so /tmp/ps_current.so
for r in $(seq ${ROUNDS:-2}); do
  for f in abvar/*.so; do
    cp "$f" paper_2405_08578_b200/libpeakstitch_b200.so
    echo -n "$f: "
    python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-match --no-stitch --no-pairs --no-composite 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels']['describe_kernel']['ms'])"
  done
done
cp /tmp/ps_current.so paper_2405_08578_b200/libpeakstitch_b200.so
