#!/bin/bash
# quick GPU check: parity sweep + c3f/c3/c2 bench lines (value, ms/step, roofline frac)
python tools/gpu_try.py 2>&1 | grep -E "first|advance|rror"
for c in c3f c3 c2; do
python bench.py --steps 200 --warmup 5 --config $c --no-cpu-baseline --e2e-steps 5 "$@" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '%.3e'%d['value'], '%.3f ms'%d['ms_per_step'], 'frac', d['roofline']['frac'])"
done
