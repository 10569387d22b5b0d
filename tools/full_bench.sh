#!/bin/bash
# Round-end style evidence: bench lines (ours + reference arm), ncu launch list.
set -x
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python bench.py --config c3f --no-cpu-baseline > gpurun_out/bench_c3f.json 2>&1
timeout 300 python bench.py --config c2 --no-cpu-baseline --steps 2000 > gpurun_out/bench_c2.json 2>&1
timeout 300 python bench.py --config c1 --no-cpu-baseline --steps 2000 > gpurun_out/bench_c1.json 2>&1
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 2 --fast"
timeout 300 $CMD > gpurun_out/launch_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/launch_ncu.log 2>&1
tail -c 1500 gpurun_out/bench_c3.json; tail -c 800 gpurun_out/bench_ref.json
