mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu5.log
tail -n 2 gpurun_out/pytest_gpu5.log
bash tools/ab.sh c3 c3f -- base fric1 minb4 > gpurun_out/ab5.txt 2>&1
cat gpurun_out/ab5.txt
