set -x

python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?; tail -5 gpurun_out/build.log
timeout 900 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
cat gpurun_out/bench_c2.json; tail -3 gpurun_out/bench_c2.err
bash tools/gpu_launches.sh
