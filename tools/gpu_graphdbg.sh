RSVD_GRAPH_DEBUG=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | grep -E "graph capture|metric" | cut -c1-300 | head -8
RSVD_GRAPHS=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nographs', d['value'], d['ms_per_step'])"
