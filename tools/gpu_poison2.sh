for P in none 0 63; do
  echo "== poison $P"
  if [ $P = none ]; then timeout 300 python tools/poison_probe.py bench 2>&1 | tail -8; else RSVD_POISON=$P timeout 300 python tools/poison_probe.py bench 2>&1 | tail -8; fi
done
