#!/bin/bash
# tools/c5_exact_ab.sh <reps> -- <variants>: C5 (early exit) exact-mode A/B of library builds, 300 steps
reps=$1; shift; shift
for r in $(seq $reps); do for v in "$@"; do
SWE_ABI_LENIENT=1 SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_$v.so timeout 300 python bench.py --config c5 --steps 300 --warmup 5 --no-cpu-baseline --no-parity --e2e-steps 2 --exact 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$r c5 exact $v', '%.4f ms'%d['ms_per_step'], d['activity']['active_fraction'])" || echo "$v failed"
done; done
