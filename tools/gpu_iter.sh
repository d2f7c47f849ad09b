#!/bin/bash
# Iteration pass: fast-path parity tests, HD T=25 vs oracle diag, bench (no CPU leg).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fastpath.py tests/test_gpu_engine.py -x -q > gpurun_out/pytest_fast.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fast.log
EVS_PATH=bucket timeout 600 python tools/diag3.py > gpurun_out/diag3.txt 2>&1
timeout 600 python bench.py --cpu-seconds 0 --compare-t1 0 > gpurun_out/bench.json 2> gpurun_out/bench.err
