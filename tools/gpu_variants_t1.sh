#!/bin/bash
# One-frame-per-call latency (bench per_frame_launch) of each variants/*.so.
mkdir -p gpurun_out
for v in variants/*.so; do
  cp "$v" paper_2602_15018_b200/libevsim_b200.so
  timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 0 > gpurun_out/bench_t1v.json 2> gpurun_out/bench_t1v.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_t1v.json')); p=d['per_frame_launch']
print('$v', round(p['frames_per_s']), round(p['one_step_after_the_other']['frames_per_s']), round(p['pixel_major_order']['frames_per_s']), round(d['value']))" || tail -3 gpurun_out/bench_t1v.err
done
