for t in $(grep -o "^def test_[a-z0-9_]*" tests/test_gpu_parity.py | sed 's/def //'); do
  r=$(timeout 300 python -m pytest "tests/test_gpu_parity.py::$t" "tests/test_gpu_configs.py::test_config_parity[C2]" -q -m gpu 2>&1 | tail -1)
  echo "$t :: $r"
done
