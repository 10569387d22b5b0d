mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cli.py -x -q > gpurun_out/pytest_cli.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cli.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu9.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu9.log
tail -n 30 gpurun_out/pytest_cli.log; tail -n 3 gpurun_out/pytest_gpu9.log
