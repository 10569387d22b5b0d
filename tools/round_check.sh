#!/bin/bash
# One GPU call: parity suite, headline bench + reference arm, launch list, one ncu --set full capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
bash tools/full_bench.sh
bash tools/ncu_full.sh c3 fast c3_fast
tail -3 gpurun_out/pytest_gpu.log
