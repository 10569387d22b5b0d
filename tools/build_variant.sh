#!/bin/bash
# build an experimental variant of libswe_cuda.so: tools/build_variant.sh <name> <extra nvcc flags...>
set -e
name=$1; shift
out=build/var_$name; mkdir -p $out
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden"
objs=""
for e in 1 0; do for k in 0 1 2 3; do
$NV -fmad=false -DSWE_EXACT_TU=$e -DSWE_PART=$k "$@" -c paper_1309_1230_b200/csrc/swe_step_inst.cu -o $out/s${e}${k}.o &
objs="$objs $out/s${e}${k}.o"
done; done
for e in 1 0; do for k in 0 1; do
$NV -fmad=false -DSWE_EXACT_TU=$e -DSWE_SMOOTH=$k "$@" -c paper_1309_1230_b200/csrc/swe_multi_inst.cu -o $out/m${e}${k}.o &
objs="$objs $out/m${e}${k}.o"
done; done
for f in swe_capi swe_aux swe_transport; do
$NV -fmad=false "$@" -c paper_1309_1230_b200/csrc/$f.cu -o $out/$f.o &
objs="$objs $out/$f.o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1309_1230_b200/lib/libswe_cuda_$name.so $objs -lcudart -ldl
echo built paper_1309_1230_b200/lib/libswe_cuda_$name.so
