mkdir -p gpurun_out
SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_bf.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_early_exit.py -x -q > gpurun_out/pytest_bf.log 2>&1; echo "bf rc=$?" >> gpurun_out/pytest_bf.log
tail -n 2 gpurun_out/pytest_bf.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu13.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu13.log
tail -n 2 gpurun_out/pytest_gpu13.log
bash tools/ab.sh c3 c3f d8k -- base bf 2>&1
for c in c1 c2; do timeout 120 python bench.py --steps 3000 --warmup 20 --config $c --no-cpu-baseline --e2e-steps 2 --fast 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', '%.4f ms'%d['ms_per_step'])"; done
