#!/bin/bash
# All bench configs on one GPU (short runs) + the reference arm of config 2.
mkdir -p gpurun_out
for c in 2 1 3 4 5; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-40} --warmup 3 --compare-t1 0 --cpu-seconds ${CPUS:-0} > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  echo "config $c rc=$?"; tail -c 600 gpurun_out/bench_c$c.json; tail -3 gpurun_out/bench_c$c.err
done
