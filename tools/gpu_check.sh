#!/bin/bash
# One gpurun pass: GPU parity tests, smoke, bench, launch list, ncu full of the top kernels.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 60 -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --compare-t1 0 --cpu-seconds 0 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_generate|k_tile_order" -s 8 -c 2 -o gpurun_out/prof python bench.py --steps 4 --warmup 3 --compare-t1 0 --cpu-seconds 0 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
