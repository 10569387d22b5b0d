mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_early_exit.py -x -q > gpurun_out/pytest_gpu7.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu7.log
tail -n 2 gpurun_out/pytest_gpu7.log
bash tools/ab.sh c3 c3f d8k -- base carry minb4 > gpurun_out/ab7.txt 2>&1
cat gpurun_out/ab7.txt
