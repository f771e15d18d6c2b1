echo "== hash default"; timeout 120 python tools/pass_hash.py
echo "== hash inkernel"; RSVD_SK_INKERNEL=1 timeout 120 python tools/pass_hash.py
for ms in 8 4 2 1; do echo "== ms=$ms"; RSVD_SK_MIN_SLICES=$ms RSVD_PROBE_PASS=1 timeout 120 python tools/ncu_pass.py C1 2>&1 | grep "^pass" | cut -c1-140; done
for ms in 8 4 2 1; do RSVD_SK_MIN_SLICES=$ms timeout 120 python tools/pass_sweep.py C1 2>&1 | tail -1 | sed "s/^/C1 ms=$ms /"; done
for ms in 8 2; do RSVD_SK_MIN_SLICES=$ms timeout 120 python tools/pass_sweep.py C2 2>&1 | tail -1 | sed "s/^/C2 ms=$ms /"; done
RSVD_SK_INKERNEL=1 timeout 120 python tools/pass_sweep.py C2 2>&1 | tail -1 | sed "s/^/C2 inkernel /"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -1
