mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu8.log
tail -n 3 gpurun_out/pytest_gpu8.log
