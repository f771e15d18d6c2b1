set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_diag.py -q -x --timeout 600 2>&1 | tail -15
timeout 600 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err; echo bench_C1=$?
cat gpurun_out/bench_C1.json; tail -3 gpurun_out/bench_C1.err
