#!/bin/bash
# One full measurement pass: GPU parity tests, smoke, bench (default + reference arm + all
# configs), launch list and ncu --set full of the step kernels (short runs; numbers under ncu
# are not bench values).
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in 1 3 4 5; do
  timeout 900 python bench.py --config $c --steps 40 --warmup 3 --cpu-seconds 15 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_prologue|k_generate|k_group_hist|k_tilescan|k_tile_order" -s 30 -c 50 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --compare-t1 0 --cpu-seconds 0 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_generate|k_group_hist|k_tilescan|k_tile_order" -s 12 -c 4 -o gpurun_out/prof python bench.py --steps 4 --warmup 3 --compare-t1 0 --cpu-seconds 0 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; ls -la gpurun_out
