#!/bin/bash
# for each library variant: parity sweep (exact must be bit-identical) + c3f/c3 timings in both modes
for v in "$@"; do
export SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_$v.so
echo "== $v"; timeout 300 python tools/gpu_try.py 2>&1 | grep -E "first|rror" | grep -v "mismatch None" ; echo "parity-check-done"
for c in c3f c3; do for m in "--exact" "--fast"; do
timeout 120 python bench.py --steps 100 --warmup 3 --config $c --no-cpu-baseline --e2e-steps 2 $m | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c $m', '%.3f ms'%d['ms_per_step'], 'frac', d['roofline']['frac'])"
done; done; done
