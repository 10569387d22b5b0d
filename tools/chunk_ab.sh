#!/bin/bash
# work-item geometry A/B (env hooks of guided_chunks): "c1 c2 bigpct" triples, config $1 (default c3)
c=${1:-c3}
for r in 1 2; do for cfg in "64 16 80" "62 14 80" "66 18 80" "96 24 80" "94 22 80" "98 26 80" "80 20 80" "112 28 80" "96 16 85" "96 32 75"; do
set -- $cfg
SWE_CHUNK1=$1 SWE_CHUNK2=$2 SWE_BIGPCT=$3 timeout 120 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-parity --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$r $c chunks $cfg', '%.4f ms'%d['ms_per_step'])"
done; done
