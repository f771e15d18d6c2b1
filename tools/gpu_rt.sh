python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in C1 C2; do for rt in 0 1; do
  RSVD_STAGE2_RT=$rt RSVD_PROBE_FQ=1 timeout 120 python tools/trace_step.py $c 1 2>&1 | grep -E "jacobi_svd" | sort | uniq -c | sed "s/^/$c rt=$rt /"
  RSVD_STAGE2_RT=$rt timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c rt=$rt', round(d['value'],1), round(d['ms_per_step']*1e3,1))"
done; done
RSVD_STAGE2_RT=1 timeout 1200 python -m pytest tests -q -m gpu --timeout 600 -x 2>&1 | tail -3
