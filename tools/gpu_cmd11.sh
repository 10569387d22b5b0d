mkdir -p gpurun_out
bash tools/full_bench.sh
bash tools/ncu_full.sh c3 fast c3_fast
timeout 600 python bench.py --config c5 --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_c5.json 2>&1
timeout 900 python bench.py --config c4 --steps 60 --warmup 3 > gpurun_out/bench_c4.json 2>&1
