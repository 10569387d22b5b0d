#!/bin/bash
# tools/c5_ab.sh <reps> -- <variants>: C5 (early exit) fast-mode A/B of library builds, 300 steps
reps=$1; shift; shift
for r in $(seq $reps); do for v in "$@"; do
SWE_ABI_LENIENT=1 SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_$v.so timeout 300 python bench.py --config c5 --steps 300 --warmup 5 --no-cpu-baseline --no-parity --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$r c5 $v', '%.4f ms'%d['ms_per_step'], d['activity']['active_fraction'], d['roofline']['frac'], d['clocks'].get('sm_mhz'))" || echo "$v failed"
done; done
