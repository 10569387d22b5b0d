#!/bin/bash
# Round-end evidence (one GPU call): the driver-style headline line + reference arm,
# every secondary config, the launch list of the headline command.
mkdir -p gpurun_out/bench_r2
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_r2/bench_c3.json 2> gpurun_out/bench_r2/bench_c3.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_r2/bench_ref.json 2>&1
timeout 900 python bench.py --gpus 1 --steps 600 --warmup 10 --no-cpu-baseline --no-parity --e2e-steps 2 --fast > gpurun_out/bench_r2/bench_c3_600.json 2>&1
for c in c1 c2; do timeout 300 python bench.py --config $c --steps 2000 --warmup 20 --no-cpu-baseline --no-parity > gpurun_out/bench_r2/bench_$c.json 2>&1; done
for c in c3f d8k; do timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --no-parity > gpurun_out/bench_r2/bench_$c.json 2>&1; done
timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline --no-parity > gpurun_out/bench_r2/bench_c4.json 2>&1
timeout 600 python bench.py --config c5 --steps 300 --warmup 5 --no-cpu-baseline --no-parity > gpurun_out/bench_r2/bench_c5.json 2>&1
for f in gpurun_out/bench_r2/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f'.split('/')[-1], round(d['ms_per_step'],5), d.get('roofline',{}).get('frac'), (d.get('other_mode') or {}).get('ms_per_step'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'))
" 2>/dev/null || echo "$f failed"; done
# launch list of the headline command (cold, serialised: shares, not absolute times)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/bench_r2/launches_c3.csv python bench.py --steps 20 --warmup 5 --fast --no-cpu-baseline --no-parity --e2e-steps 2 > gpurun_out/bench_r2/launches_c3.log 2>&1
python tools/launch_summary.py gpurun_out/bench_r2/launches_c3.csv "python bench.py --steps 20 --warmup 5 --fast --no-cpu-baseline --no-parity --e2e-steps 2" > gpurun_out/bench_r2/launches_c3_summary.txt 2>&1
