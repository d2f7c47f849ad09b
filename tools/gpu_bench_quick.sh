#!/bin/bash
# Short bench (no CPU baseline, no per-frame comparison): stage split per step.
mkdir -p gpurun_out
timeout 600 python bench.py --cpu-seconds 0 --compare-t1 0 "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); r=d['roofline']
print('value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'frac', round(r['frac'],4)); print({k: round(v,4) for k,v in r['stage_ms_per_step'].items()}); print('e2e', d.get('e2e',{}).get('value'))" || tail -20 gpurun_out/bench.err
