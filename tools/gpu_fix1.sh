timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "waits_for_inputs" 2>&1 | tail -2
RSVD_B200_LIB=$PWD/build/libold/librsvd_b200.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "waits_for_inputs" 2>&1 | grep -E "^E |passed|failed" | head -3
echo "== probe2 C1 C2"; timeout 300 python tools/poison_probe2.py 2>&1 | tail -2
echo "== probe2 poison 0"; RSVD_POISON=0 timeout 300 python tools/poison_probe2.py 2>&1 | tail -2
echo "== tiny poison 0 stages"; RSVD_ARENA_TINY=1 RSVD_POISON=0 timeout 300 python tools/poison_probe.py bench 2>&1 | tail -9
echo "== tiny poison 63 stages"; RSVD_ARENA_TINY=1 RSVD_POISON=63 timeout 300 python tools/poison_probe.py bench 2>&1 | tail -9
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -4 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo bench=$?
cat gpurun_out/bench_C2.json; tail -3 gpurun_out/bench_C2.err
timeout 600 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err; echo bench_C1=$?
cat gpurun_out/bench_C1.json
