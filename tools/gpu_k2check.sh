python -m pytest tests/test_gpu_fastpath.py tests/test_gpu_engine.py -x -q 2>&1 | tail -1
for i in 1 2 3; do python bench.py --cpu-seconds 0 --compare-t1 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['roofline']['stage_ms_per_step'].items()})"; done
python tools/diag_t1.py | tail -1
