timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "mixed_lengths" 2>&1 | grep -E "^E |passed|failed" | head -8
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "gaussian" 2>&1 | grep -E "^E |passed|failed" | head -8
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -k "gaussian or C2" 2>&1 | grep -E "^E |passed|failed" | head -8
