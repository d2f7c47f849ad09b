#!/bin/bash
# GPU parity suite (optionally a subset: tools/gpu_tests.sh tests/test_x.py ...)
mkdir -p gpurun_out
timeout 1500 python -m pytest ${@:-tests} -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
