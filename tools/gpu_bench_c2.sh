make -C paper_2402_17794_b200/csrc -s
timeout 300 python tools/trace_step.py C2 5 > gpurun_out/trace_c2.txt 2>&1; head -14 gpurun_out/trace_c2.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print(d['ms_per_step'],d['value'],d['e2e']['value'],d['roofline']['frac'],d['gpu_launches'])"
