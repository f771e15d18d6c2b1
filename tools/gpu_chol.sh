RSVD_PROBE_FQ=1 timeout 300 python tools/trace_step.py C2 1 2>&1 | grep -A1 "cholqr_fused" | head -4
for c in C1 C2; do timeout 600 python tools/trace_step.py $c 3 2>&1 | head -4; done
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
grep -E "^FAILED|passed|failed" gpurun_out/gpu_tests.log | head
for c in C2 C1; do
timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$c', round(d['value'],1), d['ms_per_step'])"
done
