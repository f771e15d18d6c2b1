python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in C2 C1; do for v in 0 9 10 11 5; do
  RSVD_PASS25_NN=$v RSVD_PASS25_TN=$v timeout 120 python tools/pass_sweep.py $c 2>&1 | tail -1 | sed "s/^/$c /"
done; done
