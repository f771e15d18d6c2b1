timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trials.py tests/test_gpu_edges.py -q -m gpu -k "gaussian or rng or trials or continuation" > gpurun_out/gt.log 2>&1; echo tests=$?; tail -1 gpurun_out/gt.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mt_jump --csv python tools/trace_step.py C2 1 2>/dev/null | grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.]*"' | head -3
for i in 1 2; do
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('C2', round(d['value'],1), d['ms_per_step'])"
done
