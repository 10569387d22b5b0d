#!/bin/bash
# tools/ab.sh <cfg list> -- <variants>: A/B of library builds (libswe_cuda_<v>.so), 2 repeats each,
# with the median SM clock and throttle reasons seen during each timed run
cfgs=(); while [ "$1" != "--" ]; do cfgs+=("$1"); shift; done; shift
for r in 1 2; do for c in "${cfgs[@]}"; do for m in --fast --exact; do for v in "$@"; do
SWE_ABI_LENIENT=1 SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_$v.so timeout 120 python bench.py --steps 600 --warmup 20 --config $c --no-cpu-baseline --no-parity --e2e-steps 2 $m 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['clocks']; print('$r $c $m $v', '%.4f ms'%d['ms_per_step'], k.get('sm_mhz'), ','.join(k.get('reasons', [])))" 2>/dev/null || echo "$v $c $m failed"
done; done; done; done
