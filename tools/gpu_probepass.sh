for ms in 8 2; do echo "== ms=$ms"; RSVD_SK_MIN_SLICES=$ms RSVD_PROBE_PASS=1 timeout 120 python tools/ncu_pass.py C1 2>&1 | grep "^pass" ; done
echo "== scan"; RSVD_PROBE_PASS=1 timeout 120 python tools/pass_scan.py 2>&1 | grep "^pass" | awk 'NR%2==1' | head -12
echo "== C2"; RSVD_PROBE_PASS=1 timeout 120 python tools/ncu_pass.py C2 2>&1 | grep "^pass"
