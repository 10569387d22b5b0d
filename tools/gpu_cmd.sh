mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
bash tools/full_bench.sh
bash tools/ncu_full.sh c3 fast c3_fast
timeout 600 python bench.py --config c5 --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c5.json 2>&1
timeout 900 python bench.py --config c4 --steps 60 --warmup 3 > gpurun_out/bench_c4.json 2>&1
timeout 300 python bench.py --config d8k --steps 600 --warmup 20 --no-cpu-baseline > gpurun_out/bench_d8k.json 2>&1
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
