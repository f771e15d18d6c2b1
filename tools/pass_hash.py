"""Bit pattern hash of apply/adjoint results at C1/C2 shapes (A/B of pass
schedules: results must be bitwise identical)."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17794_b200 as eng  # noqa: E402
from tools.pass_bench import SHAPES  # noqa: E402

for c in ("C1", "C2", "C3"):
    m, n, l = SHAPES[c]
    if c == "C3":
        m, n = 16384, 4096
    torch.manual_seed(0)
    a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    x = torch.randn(l, n, dtype=torch.float64, device="cuda").t()
    y = torch.randn(l, m, dtype=torch.float64, device="cuda").t()
    h = hashlib.sha1(eng.apply(a, x).cpu().numpy().tobytes() + eng.apply_adjoint(a, y).cpu().numpy().tobytes())
    print(c, h.hexdigest()[:16])
