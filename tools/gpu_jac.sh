RSVD_PROBE_FQ=1 timeout 300 python tools/trace_step.py C1 1 2>&1 | grep -A1 "jacobi_svd" | head -2
RSVD_PROBE_FQ=1 timeout 300 python tools/trace_step.py C2 1 2>&1 | grep "jacobi_svd" | head -1
for c in C1 C2; do timeout 600 python tools/trace_step.py $c 3 2>&1 | head -5; done
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
grep -E "^FAILED|passed|failed" gpurun_out/gpu_tests.log | head
