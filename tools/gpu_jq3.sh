RSVD_PROBE_FQ=1 timeout 300 python tools/trace_step.py C2 1 2>&1 | grep "jacobi_svd" | head -1
RSVD_PROBE_FQ=1 timeout 300 python tools/trace_step.py C1 1 2>&1 | grep "jacobi_svd" | head -1
RSVD_PROBE_FQ=1 timeout 300 python tools/trace_step.py C3 1 2>&1 | grep "bjacobi" | head -1
RSVD_PROBE_FQ=1 timeout 300 python tools/trace_step.py C4 1 2>&1 | grep "bjacobi" | head -2
for c in C1 C2 C3 C4; do timeout 600 python tools/trace_step.py $c 3 > gpurun_out/trace_$c.txt 2>&1; head -4 gpurun_out/trace_$c.txt; done
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
grep -E "^FAILED|passed|failed" gpurun_out/gpu_tests.log | head
