SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_e32.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_strips.py -x -q 2>&1 | tail -2
bash tools/ab.sh c3 c3f d8k -- base e32 2>&1 | grep fast
