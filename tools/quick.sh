#!/bin/bash
# quick GPU check: parity sweep + bench lines (value, ms/step, roofline frac) in both modes
timeout 300 python tools/gpu_try.py 2>&1 | grep -E "first|advance|rror|FAST"
for c in c3f c3 c2; do
for m in "--exact" "--fast"; do
timeout 120 python bench.py --steps 200 --warmup 5 --config $c --no-cpu-baseline --e2e-steps 5 $m "$@" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $m', '%.3e'%d['value'], '%.3f ms'%d['ms_per_step'], 'frac', d['roofline']['frac'])"
done
done
