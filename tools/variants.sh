#!/bin/bash
# time c3f/c3 (exact, fast) for each library variant given on the command line
for v in "$@"; do
for c in c3f c3; do for m in "" "--fast"; do
SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_$v.so timeout 120 python bench.py --steps 100 --warmup 3 --config $c --no-cpu-baseline --e2e-steps 2 $m | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c $m', '%.3f ms'%d['ms_per_step'], 'frac', d['roofline']['frac'])"
done; done; done
