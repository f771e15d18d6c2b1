set -x
for L in build/libold/librsvd_b200.so paper_2402_17794_b200/lib/librsvd_b200.so; do
  RSVD_B200_LIB=$PWD/$L timeout 600 python tools/debug_c2_angle.py 0 bench 2>&1 | tail -8
  RSVD_B200_LIB=$PWD/$L timeout 600 python -m pytest tests/test_gpu_configs.py -q -m gpu -k "C1 or C2" 2>&1 | grep -E "assert|passed|failed" | head -5
done
