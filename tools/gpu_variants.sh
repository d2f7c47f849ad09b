#!/bin/bash
# Bench each variants/*.so in turn (copied over the in-tree library): quick A/B of kernel variants.
for v in variants/*.so; do
  cp "$v" paper_2602_15018_b200/libevsim_b200.so
  echo "== $v"; bash tools/gpu_bench_quick.sh "$@" | head -2
done
