for i in 1 2; do for E in 0 1; do
if [ $E = 1 ]; then export RSVD_SK_INKERNEL=1; else unset RSVD_SK_INKERNEL; fi
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('inkernel=$E C2', round(d['value'],1), d['ms_per_step'], d['passes']['apply']['ms_per_launch'], d['passes']['adjoint']['ms_per_launch'])"
timeout 600 python bench.py --config C1 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('inkernel=$E C1', round(d['value'],1), d['ms_per_step'], d['passes']['apply']['ms_per_launch'], d['passes']['adjoint']['ms_per_launch'])"
done; done
