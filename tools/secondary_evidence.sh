#!/bin/bash
# Bench lines of the secondary configs (C1, C2, C3f, d8k, C4, C5) and launch lists of C2 / C5.
mkdir -p gpurun_out
for c in c1 c2; do timeout 300 python bench.py --config $c --steps 2000 --warmup 20 --no-cpu-baseline --no-parity > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
for c in c3f d8k; do timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --no-parity > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline --no-parity > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c5 --steps 300 --warmup 5 --no-cpu-baseline --no-parity > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c2 c5; do
  CMD="python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 2 --fast"
  timeout 300 $CMD > gpurun_out/launch_plain_$c.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_$c.csv $CMD > gpurun_out/launch_ncu_$c.log 2>&1
done
for c in c1 c2 c3f d8k c4 c5; do python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],5), d['roofline']['frac'], d['other_mode']['ms_per_step'] if d.get('other_mode') else '', d['clocks'].get('sm_mhz'))" 2>/dev/null || echo "$c failed"; done
