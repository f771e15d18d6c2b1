echo "== tiny, no poison: stages"; RSVD_ARENA_TINY=1 timeout 300 python tools/poison_probe.py bench 2>&1 | tail -8
echo "== tiny, poison 63: stages"; RSVD_ARENA_TINY=1 RSVD_POISON=63 timeout 300 python tools/poison_probe.py bench 2>&1 | tail -8
echo "== tiny, poison 0: stages"; RSVD_ARENA_TINY=1 RSVD_POISON=0 timeout 300 python tools/poison_probe.py bench 2>&1 | tail -8
