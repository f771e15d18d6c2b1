python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2; do
  for v in 0 9; do
    RSVD_PASS25_NN=$v RSVD_PASS25_TN=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v$v', round(d['value'],1), round(d['ms_per_step'],4), round(d['passes']['apply']['ms_per_launch']*1e3,1), round(d['passes']['adjoint']['ms_per_launch']*1e3,1))"
  done
done
