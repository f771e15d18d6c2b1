# C1 pass sweep: stream-K min slices x kernel variant, L2 flushed and warm
set -x
for ms in 8 4 3 2 1; do for v in 0 9 11; do
  RSVD_SK_MIN_SLICES=$ms RSVD_PASS25_NN=$v RSVD_PASS25_TN=$v timeout 120 python tools/pass_sweep.py C1 2>&1 | tail -1 | sed "s/^/ms=$ms /"
  NOFLUSH=1 RSVD_SK_MIN_SLICES=$ms RSVD_PASS25_NN=$v RSVD_PASS25_TN=$v timeout 120 python tools/pass_sweep.py C1 2>&1 | tail -1 | sed "s/^/warm ms=$ms /"
done; done
