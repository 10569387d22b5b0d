mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_strips.py -x -q > gpurun_out/pytest_strips.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_strips.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu4.log
tail -n 3 gpurun_out/pytest_strips.log gpurun_out/pytest_gpu4.log
