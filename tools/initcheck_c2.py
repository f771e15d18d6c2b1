"""One C2-shaped rsvd (Alg 3, 8192^2, k 20 p 5 q 2) on a fresh handle, for
compute-sanitizer --tool initcheck (reads of never-written workspace)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17794_b200 as eng  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda").t()
f = eng.rsvd(a, eng.SketchConfig(20, 5, 2, eng.RangeMode.power, 1))
torch.cuda.synchronize()
print("sigma", f.sigma[:3].cpu().numpy())
