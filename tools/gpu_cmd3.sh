mkdir -p gpurun_out
CMD="python tools/prof_step.py c5 40 fast"
timeout 300 $CMD > gpurun_out/c5_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 40 --csv --log-file gpurun_out/c5_launches.csv $CMD > gpurun_out/c5_ncu.log 2>&1
tail -n 2 gpurun_out/c5_plain.log gpurun_out/c5_ncu.log
