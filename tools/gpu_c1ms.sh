for r in 1 2; do for ms in 8 4 2; do
  RSVD_SK_MIN_SLICES=$ms timeout 300 python bench.py --config C1 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms=$ms', round(d['value'],1), round(d['ms_per_step']*1e3,1), round(d['passes']['apply']['ms_per_launch']*1e3,1), round(d['passes']['adjoint']['ms_per_launch']*1e3,1))"
done; done
