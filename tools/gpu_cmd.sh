timeout 900 python -m pytest tests/test_gpu_strips.py tests/test_gpu_cli.py -x -q > gpurun_out/pytest_last.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_last.log
tail -n 4 gpurun_out/pytest_last.log
