#!/bin/bash
# A/B of variants/*.so on one bench config (short run): CFG=1 bash tools/gpu_variants_cfg.sh
mkdir -p gpurun_out
for v in variants/*.so; do
  cp "$v" paper_2602_15018_b200/libevsim_b200.so
  timeout 600 python bench.py --config ${CFG:-1} --steps ${STEPS:-40} --warmup 3 --compare-t1 0 --cpu-seconds 0 > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); r=d['roofline']
print('$v', round(d['value']), 'ms', round(d['ms_per_step'],4), {k: round(v,4) for k,v in r['stage_ms_per_step'].items()})" || tail -5 gpurun_out/bench_v.err
done
