mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu6.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu6.log
tail -n 3 gpurun_out/pytest_gpu6.log
timeout 900 python bench.py --config c4 --steps 100 --warmup 5 > gpurun_out/b6_c4.json 2> gpurun_out/b6_c4.err
tail -c 1500 gpurun_out/b6_c4.json; tail -n 5 gpurun_out/b6_c4.err
free -g | head -2
