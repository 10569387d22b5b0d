#!/bin/bash
# small-grid item height A/B (SWE_SMALL_CHUNK rows per item; default: 4-16 by worker count)
for r in 1 2; do for c in c1 c2; do for ch in def 4 8 12 16; do
if [ $ch = def ]; then unset SWE_SMALL_CHUNK; else export SWE_SMALL_CHUNK=$ch; fi
timeout 300 python bench.py --config $c --steps 2000 --warmup 20 --no-cpu-baseline --no-parity --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$r $c chunk=$ch', '%.2f us/step'%(1e3*d['ms_per_step']), 'exact %.2f us'%(1e3*d['other_mode']['ms_per_step']))" || echo "$c $ch failed"
done; done; done
