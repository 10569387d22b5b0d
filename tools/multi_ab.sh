#!/bin/bash
# multi-step launches (small grids) vs one launch per step
for r in 1 2; do for c in c1 c2; do for m in 1 0; do
SWE_MULTI=$m timeout 300 python bench.py --config $c --steps 2000 --warmup 20 --no-cpu-baseline --no-parity --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$r $c multi=$m', '%.2f us/step'%(1e3*d['ms_per_step']), 'exact %.2f us'%(1e3*d['other_mode']['ms_per_step']), d['gpu_launches'])" || echo "$c $m failed"
done; done; done
