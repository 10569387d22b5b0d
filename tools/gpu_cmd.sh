mkdir -p gpurun_out
bash tools/full_bench.sh
bash tools/ncu_full.sh c3 fast c3_fast
