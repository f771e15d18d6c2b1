set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for ms in 8 4 2 1; do for v in 0 5 8; do RSVD_SK_MIN_SLICES=$ms RSVD_PASS25_NN=$v RSVD_PASS25_TN=$v timeout 120 python tools/pass_sweep.py C1 2>&1 | tail -1 | sed "s/^/ms=$ms /"; done; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pass_kernel -c 2 -o gpurun_out/prof_pass_C1 python tools/ncu_pass.py C1 > gpurun_out/ncu_c1full.log 2>&1; echo ncu=$?
