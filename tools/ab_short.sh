#!/bin/bash
# tools/ab_short.sh <reps> <steps> <cfg list> -- <variants>: fast-mode A/B of library builds at the
# driver's short timed region (power headroom intact for short runs)
reps=$1; shift; steps=$1; shift
cfgs=(); while [ "$1" != "--" ]; do cfgs+=("$1"); shift; done; shift
for r in $(seq $reps); do for c in "${cfgs[@]}"; do for v in "$@"; do
SWE_ABI_LENIENT=1 SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_$v.so timeout 120 python bench.py --steps $steps --warmup 5 --config $c --no-cpu-baseline --no-parity --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['clocks']; print('$r $c $v', '%.4f ms'%d['ms_per_step'], k.get('sm_mhz'), ','.join(k.get('reasons', [])))" 2>/dev/null || echo "$v $c failed"
done; done; done
