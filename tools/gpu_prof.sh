#!/bin/bash
# ncu --set full of the step kernels on the default bench workload (short run; numbers under
# ncu are not bench values), plus the launch list of the same command.
mkdir -p gpurun_out
K=${KERNELS:-k_generate|k_group_hist|k_tile_order}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 12 -c ${COUNT:-3} -o gpurun_out/prof python bench.py --steps 4 --warmup 3 --compare-t1 0 --cpu-seconds 0 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_prologue|k_generate|k_group_hist|k_tilescan|k_tile_order" -s 30 -c 50 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --compare-t1 0 --cpu-seconds 0 > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
