echo "== tiny, poison 63: stages"; RSVD_ARENA_TINY=1 RSVD_POISON=63 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/poison_probe.py bench 2>&1 | grep -v "^  File\|^    " | head -30
echo "== tiny, poison 0: stages"; RSVD_ARENA_TINY=1 RSVD_POISON=0 timeout 300 python tools/poison_probe.py bench 2>&1 | tail -9
