# launch list of a short bench run (per-kernel device times, cold/serialised)
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo ncu=$?
