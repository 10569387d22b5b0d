timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_last.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_last.log
tail -n 4 gpurun_out/pytest_last.log
bash tools/ab.sh c3 c3f -- head xs 2>&1
