#!/bin/bash
# multi-step launch grid size A/B on C1/C2 (SWE_MULTI_CTAS)
for c in c1 c2; do for n in 37 74 148 296 0; do
if [ $n = 0 ]; then unset SWE_MULTI_CTAS; else export SWE_MULTI_CTAS=$n; fi
timeout 120 python bench.py --config $c --steps 2000 --warmup 20 --no-cpu-baseline --no-parity --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c ctas $n', '%.2f us/step'%(1e3*d['ms_per_step']))"
done; done
