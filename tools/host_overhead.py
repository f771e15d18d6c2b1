"""Host-side overhead of one eng.rsvd call at C1 (cProfile of 200 calls)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
a = bench.make_input(cfg, torch.device("cuda", 0))
sk = eng.SketchConfig(cfg["k"], cfg["p"], cfg["q"], eng.RangeMode[cfg["mode"]], 1)
for _ in range(5):
    eng.rsvd(a, sk, eng.Rng(1))
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    eng.rsvd(a, sk, eng.Rng(1))
torch.cuda.synchronize()
print(f"wall per call {(time.perf_counter() - t0) / 200 * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    eng.rsvd(a, sk, eng.Rng(1))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
