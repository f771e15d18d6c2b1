M=gpu__time_duration.sum,launch__grid_size
timeout 300 ncu --metrics $M --clock-control none --cache-control none -k regex:pass_kernel --csv python tools/pass_scan.py > gpurun_out/scan2.csv 2> gpurun_out/scan2.err
RSVD_SK_MIN_SLICES=2 timeout 300 ncu --metrics $M --clock-control none --cache-control none -k regex:pass_kernel --csv python tools/pass_scan.py > gpurun_out/scan2_ms2.csv 2>> gpurun_out/scan2.err
for ms in 8 4 2 1; do RSVD_SK_MIN_SLICES=$ms timeout 120 python tools/pass_sweep.py C1 2>&1 | tail -1 | sed "s/^/ms=$ms /"; done
for ms in 8 2; do RSVD_SK_MIN_SLICES=$ms timeout 120 python tools/pass_sweep.py C2 2>&1 | tail -1 | sed "s/^/C2 ms=$ms /"; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "apply or pass or rsvd" 2>&1 | tail -1
