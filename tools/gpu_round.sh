# Validate HEAD on a B200: build + smoke, all GPU tests, C1/C2 bench lines, launch-site traces.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build.log 2>&1; echo build_smoke=$?
tail -3 gpurun_out/build.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -8 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo bench=$?
cat gpurun_out/bench_C2.json; tail -3 gpurun_out/bench_C2.err
timeout 600 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err; echo bench_C1=$?
cat gpurun_out/bench_C1.json
for c in C1 C2 C3 C4; do timeout 600 python tools/trace_step.py $c 3 > gpurun_out/trace_$c.txt 2>&1; cat gpurun_out/trace_$c.txt | head -14; done
