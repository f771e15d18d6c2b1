python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in C3 C5s; do for v in 0 1 2; do
  RSVD_PASSBIG=$v timeout 300 python tools/pass_sweep.py $c 2>&1 | tail -1 | sed "s/^/$c big=$v /"
done; done
