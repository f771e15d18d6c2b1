"""One apply and one adjoint pass at a BASELINE shape (for ncu captures):
python tools/ncu_pass.py C2"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17794_b200 as eng  # noqa: E402
from tools.pass_bench import SHAPES  # noqa: E402

m, n, l = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "C2"]
torch.manual_seed(0)
a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
x = torch.randn(l, n, dtype=torch.float64, device="cuda").t()
y = torch.randn(l, m, dtype=torch.float64, device="cuda").t()
eng.apply(a, x)
eng.apply_adjoint(a, y)
torch.cuda.synchronize()
