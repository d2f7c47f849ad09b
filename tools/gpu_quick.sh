#!/bin/bash
# Quick GPU pass: fast-path parity tests, full GPU suite, bench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fastpath.py -x -q > gpurun_out/pytest_fast.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fast.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --cpu-seconds 0 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/pytest_fast.log gpurun_out/pytest_gpu.log
