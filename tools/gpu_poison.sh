for P in 0 255 63 17; do
  echo "poison $P"; RSVD_POISON=$P timeout 600 python -m pytest tests/test_gpu_configs.py -q -m gpu -k "C1 or C2" 2>&1 | grep -E "^E |passed|failed" | head -4
done
echo "poison 63 parity"; RSVD_POISON=63 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -m gpu 2>&1 | grep -E "^FAILED|passed|failed" | head -12
