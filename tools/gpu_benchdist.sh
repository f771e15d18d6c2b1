for c in C2 C1 C4; do
RSVD_BENCH_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bdist_$c.json 2> gpurun_out/bdist_$c.err; echo "$c rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bdist_$c.json')); print('$c', round(d['value'],2), d['ms_per_step'], d['config']['parallelism'], 'e2e', round(d['e2e']['value'],2), d['roofline']['frac'])" 2>&1 | tail -1
tail -2 gpurun_out/bdist_$c.err
done
