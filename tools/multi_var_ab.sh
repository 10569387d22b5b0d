#!/bin/bash
# tools/multi_var_ab.sh <reps> -- <variants>: small-grid (multi-step launch) A/B of library builds, fast + exact
reps=$1; shift; shift
for r in $(seq $reps); do for c in c1 c2; do for v in "$@"; do
SWE_ABI_LENIENT=1 SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_$v.so timeout 300 python bench.py --config $c --steps 2000 --warmup 20 --no-cpu-baseline --no-parity --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$r $c $v', '%.2f us/step'%(1e3*d['ms_per_step']), 'exact %.2f us'%(1e3*d['other_mode']['ms_per_step']))" || echo "$c $v failed"
done; done; done
