#!/bin/bash
# Per-kernel launch list (ncu gpu__time_duration, serialised) of each variants/*.so on a short HD bench.
mkdir -p gpurun_out
for v in variants/*.so; do
  cp "$v" paper_2602_15018_b200/libevsim_b200.so
  b=$(basename $v .so)
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_prologue|k_generate|k_group_hist|k_tilescan|k_tile_order" -s 30 -c 25 --csv --log-file gpurun_out/ll_$b.csv python bench.py --steps 10 --warmup 3 --compare-t1 0 --cpu-seconds 0 > /dev/null 2>&1
  echo "== $b"; python tools/launch_summary.py gpurun_out/ll_$b.csv | tail -6
done
