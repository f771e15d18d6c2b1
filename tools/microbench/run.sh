set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 250 > gpurun_out/mb_clocks.csv &
SMI=$!
./tools/microbench/fp64_peak > gpurun_out/mb_fp64.txt 2>&1
python tools/microbench/cublas_dgemm.py > gpurun_out/mb_cublas.txt 2>&1
kill $SMI
lscpu > gpurun_out/mb_lscpu.txt; nproc >> gpurun_out/mb_lscpu.txt; free -g >> gpurun_out/mb_lscpu.txt
cat gpurun_out/mb_fp64.txt gpurun_out/mb_cublas.txt
