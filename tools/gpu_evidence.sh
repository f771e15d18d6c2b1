# Round evidence: build + smoke, GPU tests, bench lines C1-C5 (+ reference
# arm), launch-site traces, ncu launch list + full captures of the C1/C2/C3
# passes, C5 full-size parity.  Outputs -> gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build.log 2>&1; echo build_smoke=$?
tail -2 gpurun_out/build.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo bench=$?
cat gpurun_out/bench_C2.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_C2.json 2> gpurun_out/bench_ref_C2.err; echo ref=$?
cat gpurun_out/bench_ref_C2.json
for c in C1 C3 C4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?
  cat gpurun_out/bench_$c.json
done
timeout 1500 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo bench_C5=$?
cat gpurun_out/bench_C5.json
for c in C1 C2 C3 C4 C5; do timeout 900 python tools/trace_step.py $c 2 > gpurun_out/trace_$c.txt 2>&1; done
for c in C1 C2; do for T in 10 30; do timeout 300 python tools/trials_bench.py $c $T; done; done > gpurun_out/trials_bench.txt 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo ncu1=$?
for c in C1 C2; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pass_kernel -c 2 -o gpurun_out/prof_pass_$c python tools/ncu_pass.py $c > gpurun_out/ncu_full_$c.log 2>&1; echo ncu_$c=$?
done
timeout 2400 python tools/parity_config.py C5 > gpurun_out/parity_C5.log 2>&1; echo parity_C5=$?
tail -5 gpurun_out/parity_C5.log
ls -la gpurun_out
