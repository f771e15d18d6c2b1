export RSVD_JACOBI_BLOCK=1
RSVD_PROBE_FQ=1 timeout 300 python tools/trace_step.py C1 1 2>&1 | grep "bjacobi" | head -2
RSVD_PROBE_FQ=1 timeout 300 python tools/trace_step.py C2 1 2>&1 | grep "bjacobi" | head -2
for c in C1 C2; do timeout 600 python tools/trace_step.py $c 3 2>&1 | head -5; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_edges.py -q -m gpu --timeout 600 -k "not C3 and not C4" > gpurun_out/gpu_tests_bj.log 2>&1; echo tests=$?
grep -E "^FAILED|passed|failed" gpurun_out/gpu_tests_bj.log | head
