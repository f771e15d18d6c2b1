set -x
M=gpu__time_duration.sum,launch__grid_size,sm__cycles_active.avg,sm__cycles_elapsed.avg
timeout 300 ncu --metrics $M --clock-control none --cache-control none -k regex:pass_kernel --csv python tools/pass_scan.py > gpurun_out/scan.csv 2> gpurun_out/scan.err
RSVD_SK_MIN_SLICES=1 timeout 300 ncu --metrics $M --clock-control none --cache-control none -k regex:pass_kernel --csv python tools/pass_scan.py > gpurun_out/scan_ms1.csv 2>> gpurun_out/scan.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_edges.py tests/test_gpu_diag.py -q -m gpu -x > gpurun_out/jq_tests.log 2>&1; echo tests=$?
tail -5 gpurun_out/jq_tests.log
for c in C1 C2; do timeout 600 python tools/trace_step.py $c 3 > gpurun_out/trace_$c.txt 2>&1; head -6 gpurun_out/trace_$c.txt; done
RSVD_PROBE_FQ=1 timeout 600 python tools/trace_step.py C3 1 2>&1 | grep -i "bjacobi\|C3:" | head
