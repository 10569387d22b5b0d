mkdir -p gpurun_out
for v in two two4; do
SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_early_exit.py tests/test_gpu_strips.py -x -q > gpurun_out/pytest_$v.log 2>&1; echo "$v rc=$?" >> gpurun_out/pytest_$v.log
tail -n 2 gpurun_out/pytest_$v.log
done
bash tools/ab.sh c3 c3f d8k -- base two two4 2>&1
