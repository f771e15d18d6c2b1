timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
grep -E "^FAILED|^E |passed|failed" gpurun_out/gpu_tests.log | head
for c in C1 C2 C1 C2; do
timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/bench_o.json 2> gpurun_out/bench_o.err
python -c "import json; d=json.load(open('gpurun_out/bench_o.json')); print('$c', round(d['value'],1), d['ms_per_step'], 'e2e', round(d['e2e']['value'],1), d['e2e']['ms_per_step'])"
done
