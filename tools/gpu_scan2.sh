timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
grep -E "^FAILED|passed|failed" gpurun_out/gpu_tests.log | head
for i in 1 2; do for c in C2 C1; do
timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$c', round(d['value'],1), d['ms_per_step'], d['gpu_launches'])"
done; done
