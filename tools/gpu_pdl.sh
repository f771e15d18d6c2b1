timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
grep -E "^FAILED|^E |passed|failed" gpurun_out/gpu_tests.log | head
for P in 1 0 1 0; do
RSVD_PDL=$P timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
python -c "import json; d=json.load(open('gpurun_out/bench_C2.json')); print('PDL=$P C2', round(d['value'],1), d['ms_per_step'], d['passes']['apply']['ms_per_launch'], d['passes']['adjoint']['ms_per_launch'], d['roofline']['frac'], d['profiled_run_ms_per_step'])"
RSVD_PDL=$P timeout 600 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
python -c "import json; d=json.load(open('gpurun_out/bench_C1.json')); print('PDL=$P C1', round(d['value'],1), d['ms_per_step'], d['passes']['apply']['ms_per_launch'], d['passes']['adjoint']['ms_per_launch'], d['roofline']['frac'], d['profiled_run_ms_per_step'])"
done
RSVD_GRAPH_DEBUG=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | grep -E "graph capture" | cut -c1-80
