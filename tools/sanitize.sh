#!/bin/bash
# compute-sanitizer passes over small GPU parity cases (memcheck, racecheck, synccheck),
# default path and bucket path separately
mkdir -p gpurun_out
DEF="tests/test_gpu_engine.py tests/test_gpu_golden.py tests/test_gpu_event_parallel.py"
BKT="tests/test_gpu_fastpath.py::test_fast_matches_oracle tests/test_gpu_fastpath.py::test_capacity_cut tests/test_gpu_fastpath.py::test_overflow_tiles_sorted_by_fixup"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python -m pytest $DEF -x -q > gpurun_out/sanitize_default_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_default_$tool.log
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python -m pytest $BKT -x -q > gpurun_out/sanitize_bucket_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_bucket_$tool.log
done
