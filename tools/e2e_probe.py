"""Where the e2e (host-buffer) C2 step spends its time: raw pinned H2D copy
bandwidth vs the rsvd_rsvd_host call, repeated."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402

cfg = bench.CONFIGS["C2"]
dev = torch.device("cuda", 0)
a = bench.make_input(cfg, dev)
n = a.shape[1]
pin = torch.empty((n, a.shape[0]), dtype=torch.float64, pin_memory=True)
pin.copy_(a.t())
print("pinned:", pin.is_pinned())
d = torch.empty_like(pin, device=dev)
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(pin, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"torch H2D {pin.numel() * 8 / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms)")
a_host = pin.numpy().T
sk = eng.SketchConfig(20, 5, 2, eng.RangeMode.power, 1)
for i in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.rsvd_host(a_host, sk, eng.Rng(1))
    dt = time.perf_counter() - t0
    print(f"rsvd_host {dt * 1e3:.1f} ms")
