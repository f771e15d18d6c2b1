python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python tools/probe_c2.py > gpurun_out/probe.txt 2>&1; tail -4 gpurun_out/probe.txt
timeout 300 python tools/trace_step.py C2 5 > gpurun_out/trace_c2.txt 2>&1; head -6 gpurun_out/trace_c2.txt
timeout 900 python -m pytest tests -q -m gpu -x --timeout 600 ${PYTEST_K} > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -4 gpurun_out/gpu_tests.log
