#!/bin/bash
# A/B of variants/*.so on tools/k1_split.py (static scene vs moving texture) and the quick bench.
for v in variants/*.so; do
  cp "$v" paper_2602_15018_b200/libevsim_b200.so
  echo "== $v"; python tools/k1_split.py 2>&1 | tail -2; bash tools/gpu_bench_quick.sh | head -2
done
