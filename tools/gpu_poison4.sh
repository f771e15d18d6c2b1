for P in none 0 63; do
  echo "== poison $P"
  if [ $P = none ]; then timeout 300 python tools/poison_probe2.py 2>&1 | tail -3; else RSVD_POISON=$P timeout 300 python tools/poison_probe2.py 2>&1 | tail -3; fi
done
echo "== C2 only poison 63"; RSVD_POISON=63 timeout 300 python tools/poison_probe2.py C2 2>&1 | tail -3
echo "== C2 C2 poison 63"; RSVD_POISON=63 timeout 300 python tools/poison_probe2.py C2 C2 2>&1 | tail -3
