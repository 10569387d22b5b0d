#!/bin/bash
# persistent-grid size A/B (SWE_NCTA CTAs of 4 warps): tools/ncta_ab.sh <config> <ncta list...>
c=$1; shift
for r in 1 2; do for n in "$@"; do
if [ $n = def ]; then unset SWE_NCTA; else export SWE_NCTA=$n; fi
timeout 300 python bench.py --config $c --steps 300 --warmup 5 --no-cpu-baseline --no-parity --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$r $c ncta=$n', '%.4f ms'%d['ms_per_step'])" || echo "$c $n failed"
done; done
