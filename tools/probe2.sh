#!/bin/bash
# tools/probe2.sh <cfg list> -- <variants>
cfgs=(); while [ "$1" != "--" ]; do cfgs+=("$1"); shift; done; shift
for v in "$@"; do for c in "${cfgs[@]}"; do for m in --fast --exact; do
SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_$v.so timeout 120 python bench.py --steps 100 --warmup 3 --config $c --no-cpu-baseline --e2e-steps 2 $m 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c $m', '%.3f ms'%d['ms_per_step'], 'frac', d['roofline']['frac'])" 2>/dev/null || echo "$v $c $m failed"
done; done; done
