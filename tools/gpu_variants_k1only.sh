#!/bin/bash
# K1 stage time only (tools/k1_split.py) of each variants/*.so -- for timing experiments whose output is not checked.
for v in variants/*.so; do
  cp "$v" paper_2602_15018_b200/libevsim_b200.so
  echo "== $v"; python tools/k1_split.py 2>&1 | tail -2
done
