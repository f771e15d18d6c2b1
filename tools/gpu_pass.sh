make -C paper_2402_17794_b200/csrc -s
for c in C2 C3 C4 C5s; do python tools/pass_bench.py $c 10; done
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
