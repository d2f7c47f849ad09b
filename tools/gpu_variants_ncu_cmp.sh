#!/bin/bash
# ncu --set full of one launch of $KERNELS for each variants/*.so (short HD bench); summaries side by side.
mkdir -p gpurun_out
for v in variants/*.so; do
  cp "$v" paper_2602_15018_b200/libevsim_b200.so
  b=$(basename $v .so)
  timeout 600 ncu --set full --clock-control none -k regex:"${KERNELS:-k_group_hist|k_tile_order}" -s 6 -c ${COUNT:-2} -o gpurun_out/cmp_$b python bench.py --steps 4 --warmup 3 --compare-t1 0 --cpu-seconds 0 > /dev/null 2>&1
  echo "== $b"; python tools/ncu_summary.py gpurun_out/cmp_$b.ncu-rep "$b" | grep -E "==|duration|inst_executed.sum|issue_active|warps_active|stalls"
done
