mkdir -p gpurun_out
timeout 300 python bench.py --config c5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 100 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
bash tools/ncu_full.sh c5 fast c5_fast
CMD="python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 2 --fast"
timeout 300 $CMD > gpurun_out/launch_plain_c5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/launch_ncu_c5.log 2>&1
echo rc=$?
