timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cli.py -x -q > gpurun_out/pytest_gpu17.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu17.log
tail -n 3 gpurun_out/pytest_gpu17.log
timeout 300 python bench.py --steps 600 --warmup 20 --config c3 --no-cpu-baseline --e2e-steps 2 --exact 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['clocks']; print('c3 exact', '%.4f ms'%d['ms_per_step'], d['roofline']['frac'], k.get('sm_mhz'), k.get('reasons'))"
