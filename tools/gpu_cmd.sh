timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_last.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_last.log
tail -n 2 gpurun_out/pytest_last.log
timeout 600 python bench.py --steps 300 --warmup 5 --config c5 --no-cpu-baseline --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5 fast', '%.4f ms'%d['ms_per_step'], 'exact', '%.4f'%d['other_mode']['ms_per_step'], d['activity']['active_fraction'])"
timeout 300 python bench.py --steps 600 --warmup 20 --config c3 --no-cpu-baseline --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 fast', '%.4f ms'%d['ms_per_step'])"
