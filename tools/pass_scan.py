"""Apply / adjoint passes over a range of K (= n) at m = 2048, l = 25, for
ncu per-launch durations: where does the fixed cost of a small pass go?
Usage: ncu --metrics gpu__time_duration.sum ... python tools/pass_scan.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17794_b200 as eng  # noqa: E402

m, l = int(os.environ.get("SCAN_M", "2048")), 25
for n in (48, 96, 192, 384, 1024, 4096):
    a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    x = torch.randn(l, n, dtype=torch.float64, device="cuda").t()
    y = torch.randn(l, m, dtype=torch.float64, device="cuda").t()
    for _ in range(2):
        eng.apply(a, x)
        eng.apply_adjoint(a, y)
torch.cuda.synchronize()
