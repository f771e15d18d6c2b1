make -C paper_2402_17794_b200/csrc -s
for g in 0 1; do for c in C1 C2; do echo "graphs=$g $c"; RSVD_GRAPHS=$g python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(d['ms_per_step'], d['gpu_launches'])"; done; done
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
