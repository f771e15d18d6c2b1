# C1 pass: ncu metrics at min-slices 8 / 1 (grid size vs duration), plus the dist1 tests
set -x
M=gpu__time_duration.sum,launch__grid_size,sm__cycles_active.avg,sm__cycles_elapsed.avg,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
for ms in 8 1; do
RSVD_SK_MIN_SLICES=$ms timeout 300 ncu --metrics $M --clock-control none -k regex:pass_kernel python tools/ncu_pass.py C1 > gpurun_out/c1ncu_ms$ms.txt 2>&1
RSVD_SK_MIN_SLICES=$ms timeout 300 ncu --metrics $M --clock-control none --cache-control none -k regex:pass_kernel python tools/ncu_pass.py C1 > gpurun_out/c1ncu_warm_ms$ms.txt 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pass_kernel -c 1 -o gpurun_out/prof_pass_C1 python tools/ncu_pass.py C1 > gpurun_out/ncu_c1full.log 2>&1
timeout 600 python -m pytest tests/test_gpu_dist1.py -q -m gpu > gpurun_out/dist1.log 2>&1; echo dist1=$?
tail -30 gpurun_out/dist1.log
