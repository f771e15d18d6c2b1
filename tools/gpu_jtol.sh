set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for c in C1 C2; do
  RSVD_PROBE_FQ=1 timeout 120 python tools/trace_step.py $c 1 2>&1 | grep -E "jacobi_svd|per factorization" | sort | uniq -c | head
  RSVD_JTOL_L=1 RSVD_PROBE_FQ=1 timeout 120 python tools/trace_step.py $c 1 2>&1 | grep -E "jacobi_svd|per factorization" | sort | uniq -c | head
  timeout 120 python tools/trace_step.py $c 5 2>&1 | head -4
  RSVD_JTOL_L=1 timeout 120 python tools/trace_step.py $c 5 2>&1 | head -4
done
RSVD_JTOL_L=1 timeout 900 python -m pytest tests -q -m gpu --timeout 600 -x -k "parity or config" 2>&1 | tail -3
