#!/bin/bash
# The race/memory-checker substitute (compute-sanitizer is closed on this pool):
# the SWE_CHECKED library (device assertions on stores, TMA coordinates, ring
# slots, work items; guard bands around every allocation) on every kernel
# family, each case compared with the CPU oracle.
mkdir -p gpurun_out
SWE_ABI_LENIENT=1 SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_checked.so timeout 900 \
    python tools/sanitize_cases.py "$@" > gpurun_out/checked_run.log 2>&1
echo "== rc=$?" >> gpurun_out/checked_run.log
cat gpurun_out/checked_run.log
