#!/bin/bash
# compute-sanitizer over the representation / noise / band tests (memcheck, racecheck, synccheck)
mkdir -p gpurun_out
T="tests/test_gpu_simulator.py tests/test_gpu_parity.py::test_noise_golden tests/test_gpu_bands.py::test_bands_invalid_frame_raises_first_pixel_and_keeps_state tests/test_gpu_bands.py::test_bands_device_output"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python -m pytest $T -x -q > gpurun_out/sanitize_new_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_new_$tool.log
done
