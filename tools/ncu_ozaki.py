"""One Alg-6 dual pass on the INT8 tensor cores (csrc/ozaki.cu) at a C5 row
panel's shape, for ncu captures:

  python tools/ncu_ozaki.py [m n l slices]      (default 32768 32768 550 7)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17794_b200 as eng  # noqa: E402


def main():
    d = [int(v) for v in sys.argv[1:5]]
    m, n, l, s = (d + [32768, 32768, 550, 7][len(d):])
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    a = torch.randn((n, m), dtype=torch.float64, device=dev, generator=g).t()
    oc = torch.randn((l, n), dtype=torch.float64, device=dev, generator=g).t()
    psi = torch.randn((l, m), dtype=torch.float64, device=dev, generator=g).t()
    eng.set_ozaki_slices(s)
    y, w = eng.debug_dual_pass(a, oc, psi)
    torch.cuda.synchronize()
    print("ok", float(y[0, 0]), float(w[0, 0]))


if __name__ == "__main__":
    main()
