timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trials.py tests/test_gpu_edges.py tests/test_gpu_configs.py -q -m gpu -k "gaussian or rng or trials or continuation or C1 or C2" > gpurun_out/gt.log 2>&1; echo tests=$?; tail -1 gpurun_out/gt.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mt_" --csv python tools/trace_step.py C2 1 2>/dev/null | grep -oE '"(rsvdb::[^"]*mt_[a-z_]*)[^"]*"|"gpu__time_duration.sum","[a-z]*","[0-9.]*"' | head -8
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mt_" --csv python tools/trace_step.py C1 1 2>/dev/null | grep -oE '"gpu__time_duration.sum","[a-z]*","[0-9.]*"' | head -3
for c in C2 C1 C2 C1; do
timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$c', round(d['value'],1), d['ms_per_step'])"
done
