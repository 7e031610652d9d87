#!/bin/bash
# GPU-box quick check: parity tests + short bench summary (stages: back-to-back
# device time; kernels: event-bracketed, ~5 us overhead each).
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('ms/step', round(d['ms_per_step'],4), 'Gvox/s', round(d['value']/1e9,2), 'e2e ms', round(d['e2e']['ms_per_step'],3), 'launches/step', d['launches_per_step'])
print('stages:', ', '.join(f\"{k} {v['ms_per_launch']*1e3:.1f}\" for k,v in d['stages'].items()))
print('kernels:', ', '.join(f\"{k} {v['ms_per_launch_event_bracketed']*1e3:.1f}\" for k,v in d['kernels'].items()))
"
