set -x
nvidia-smi --query-gpu=name --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -50 gpurun_out/gpu_tests.log
