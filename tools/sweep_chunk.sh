#!/bin/bash
# tools/sweep_chunk.sh: work-item sizing sweep (SWE_TUNE_* env) over configs
for combo in "2 16 1" "4 16 1" "8 16 1" "16 16 1" "4 16 0" "2 16 0" "8 4 1" "16 4 1"; do
set -- $combo
for c in c1 c2 d8k c3; do for m in --fast --exact; do
SWE_TUNE_CHUNK_MIN=$1 SWE_TUNE_CHUNK_DIV=$2 SWE_TUNE_CTA_FULL=$3 timeout 120 python bench.py --steps 100 --warmup 3 --config $c --no-cpu-baseline --e2e-steps 2 $m 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$combo $c $m', '%.4f ms'%d['ms_per_step'])" 2>/dev/null || echo "$combo $c $m failed"
done; done; done
