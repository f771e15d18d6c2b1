make -C paper_2402_17794_b200/csrc -s
python tools/pass_bench.py C2 20
ncu --set full --import-source on -k regex:pass_kernel -c 2 -o gpurun_out/ncu_c2_pass python tools/ncu_pass.py C2 > gpurun_out/ncu_c2.log 2>&1; tail -2 gpurun_out/ncu_c2.log
