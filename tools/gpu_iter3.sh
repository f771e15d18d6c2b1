# build, GPU tests, bench C2 (+launch list), bench C3
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
cat gpurun_out/bench_c2.json; tail -3 gpurun_out/bench_c2.err
bash tools/gpu_launches.sh
timeout 900 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench3=$?
cat gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
