#!/bin/bash
for v in "$@"; do for c in c3f c3; do
SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_$v.so timeout 120 python bench.py --steps 100 --warmup 3 --config $c --no-cpu-baseline --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c', '%.3f ms'%d['ms_per_step'], 'frac', d['roofline']['frac'])" 
done; done
