set -x
for L in build/libold/librsvd_b200.so paper_2402_17794_b200/lib/librsvd_b200.so; do
  RSVD_B200_LIB=$PWD/$L timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -k "not C3 and not C4" 2>&1 | grep -E "assert|passed|failed|Error" | head -8
done
RSVD_B200_LIB=$PWD/paper_2402_17794_b200/lib/librsvd_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py::test_graph_replay_matches_eager tests/test_gpu_configs.py -q -m gpu -k "replay or C2" 2>&1 | grep -E "assert|passed|failed|Error" | head -8
