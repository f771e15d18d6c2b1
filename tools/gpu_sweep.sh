set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for c in C2 C1; do for v in 0 1 2 3 4 5 6 7 8; do
  RSVD_PASS25_NN=$v RSVD_PASS25_TN=$v timeout 120 python tools/pass_sweep.py $c 2>&1 | tail -1
done; done
./tools/microbench/dmma_lds 2>&1 | tail -6
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C1.csv python bench.py --config C1 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c1.log 2>&1; echo ncu=$?
