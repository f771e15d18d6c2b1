set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?; tail -5 gpurun_out/build.log
timeout 300 python tools/probe_c2.py > gpurun_out/probe.txt 2>&1; tail -8 gpurun_out/probe.txt
timeout 300 python tools/trace_step.py C2 5 > gpurun_out/trace_c2.txt 2>&1; cat gpurun_out/trace_c2.txt
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
cat gpurun_out/bench_c2.json; tail -3 gpurun_out/bench_c2.err
