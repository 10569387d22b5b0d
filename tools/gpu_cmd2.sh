mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_early_exit.py -x -q > gpurun_out/pytest_early.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_early.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
timeout 600 python bench.py --config c5 --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 5 > gpurun_out/b2_c5.json 2>&1
timeout 200 python bench.py --config c3 --fast --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b2_c3.json 2>&1
tail -3 gpurun_out/pytest_early.log gpurun_out/pytest_gpu2.log
