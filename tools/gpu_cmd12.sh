mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k fast > gpurun_out/pytest_gpu12.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu12.log
tail -n 2 gpurun_out/pytest_gpu12.log
bash tools/ab.sh c3 c3f -- base rcp3 2>&1 | grep fast
for c in c1 c2; do for mc in 16 8 4; do
SWE_MIN_CHUNK=$mc timeout 120 python bench.py --steps 3000 --warmup 20 --config $c --no-cpu-baseline --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c minchunk=$mc', '%.4f ms'%d['ms_per_step'])"
done; done
