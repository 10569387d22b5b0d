bash tools/ncu_full.sh c3 fast c3_fast
