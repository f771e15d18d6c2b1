timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -k "not C3 and not C4" 2>&1 | grep -E "^E |passed|failed" | head -8
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -k "not C3 and not C4 and not gaussian" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -k "not C3 and not C4 and not orthonormalize and not svd_small and not evd and not solve and not joint" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -k "not C3 and not C4 and not rsvd and not spevd and not spsvd and not graph" 2>&1 | tail -1
