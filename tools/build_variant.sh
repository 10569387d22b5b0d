#!/bin/bash
# build an experimental variant of libswe_cuda.so: tools/build_variant.sh <name> <extra nvcc flags...>
set -e
name=$1; shift
out=build/var_$name; mkdir -p $out
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden"
$NV -fmad=false -DSWE_EXACT_TU=1 "$@" -c paper_1309_1230_b200/csrc/swe_step_inst.cu -o $out/e.o &
$NV -fmad=false -DSWE_EXACT_TU=0 "$@" -c paper_1309_1230_b200/csrc/swe_step_inst.cu -o $out/f.o &
$NV -fmad=false "$@" -c paper_1309_1230_b200/csrc/swe_capi.cu -o $out/c.o &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1309_1230_b200/lib/libswe_cuda_$name.so $out/e.o $out/f.o $out/c.o -lcudart -ldl
echo built paper_1309_1230_b200/lib/libswe_cuda_$name.so
