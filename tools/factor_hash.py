"""Bit pattern hash of full factorizations (C1, C2, C4) and of CholeskyQR
orthonormalizations (l = 25, the fused kernel; l = 110, the blocked one):
A/B of small-kernel changes that must leave results bitwise identical."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402


def h(*ts):
    d = hashlib.sha256()
    for t in ts:
        d.update(t.detach().contiguous().cpu().numpy().tobytes())
    return d.hexdigest()[:16]


for c in ("C1", "C2", "C4"):
    cfg = bench.CONFIGS[c]
    a = bench.make_input(cfg, torch.device("cuda", 0))
    k, p, q = cfg["k"], cfg["p"], cfg["q"]
    if c == "C4":
        r = eng.spevd_hermitian(a, k, p, eng.Rng(1))
        print(c, h(r.U, r.lambda_))
    else:
        r = eng.rsvd(a, eng.SketchConfig(k, p, q, eng.RangeMode[cfg["mode"]], 1))
        print(c, h(r.U, r.sigma, r.V))
    del a
    torch.cuda.empty_cache()
g = torch.Generator(device="cpu").manual_seed(7)
for m, l in ((8192, 25), (65536, 110)):
    y = torch.randn(m, l, generator=g, dtype=torch.float64)
    y[:, 1] = y[:, 0] + 1e-9 * y[:, 1]  # ill-conditioned: exercises the shift
    print("orth", m, l, h(eng.orthonormalize(y.cuda())))
