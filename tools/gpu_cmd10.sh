mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu10.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu10.log
tail -n 2 gpurun_out/pytest_gpu10.log
timeout 300 python tools/e2e_probe.py c3 50 2>&1 | tail -3
for r in 1 2; do for c in c3 c3f d8k; do for g in 1 0; do
SWE_GUIDED=$g timeout 120 python bench.py --steps 600 --warmup 20 --config $c --no-cpu-baseline --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['clocks']; print('$r $c guided=$g', '%.4f ms'%d['ms_per_step'], k.get('sm_mhz'), ','.join(k.get('reasons', [])))"
done; done; done
