"""The C2 sketch draw (8192 x 25 normals from Rng(1)) for ncu captures of the
RNG kernels: python tools/ncu_rng.py [n] [l]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17794_b200 as eng  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
l = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for _ in range(3):
    eng.gaussian(n, l, eng.Rng(1), device_out=True)
torch.cuda.synchronize()
