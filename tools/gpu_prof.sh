#!/bin/bash
# ncu full capture of the fast-path kernels on the default bench workload (short run)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fast_gen|k_fast_order" -s 10 -c 2 -o gpurun_out/prof_fast python bench.py --steps 3 --warmup 5 --compare-t1 0 --cpu-seconds 0 > gpurun_out/ncu_fast.log 2>&1
