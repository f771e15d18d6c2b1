"""Where does the GPU-vs-oracle top-20 subspace difference on C2 come from?
Compares range_basis Q and the final U of the GPU engine and the oracle
against the exact singular vectors of a C2-type matrix (numpy-generated)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402

oracle.set_threads(os.cpu_count())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rs = np.random.default_rng(1)


def haar(k):
    q, r = np.linalg.qr(rs.standard_normal((k, k)))
    return q * np.sign(np.diag(r))


if len(sys.argv) > 2 and sys.argv[2] == "bench":
    import bench
    At = bench.make_input(bench.CONFIGS["C2"], torch.device("cuda", 0))
    A = np.asfortranarray(At.cpu().numpy())
    n = A.shape[0]
    # exact top singular vectors of the generated A (dense SVD on the GPU)
    U = torch.linalg.svd(At, full_matrices=False)[0].cpu().numpy()
    print("generated A: top-22 sigma", torch.linalg.svdvals(At).cpu().numpy()[18:22])
else:
    U = haar(n)
    V = haar(n)
    j = np.arange(1, n + 1)
    s = np.ones(n)
    s[20:] = 1e-2 / (j[20:] - 20)
    A = np.asfortranarray((U * s) @ V.T)
    At = torch.from_numpy(A).cuda().t().contiguous().t()


def sinmax(x, y):
    return float(np.linalg.svd(y - x @ (x.T @ y), compute_uv=False)[0])


cfg = eng.SketchConfig(20, 5, 2, eng.RangeMode.power, 1)
qg = eng.range_basis(At, cfg, eng.Rng(1)).cpu().numpy()
qo = oracle.range_basis(A, 20, 5, 2, oracle.POWER, oracle.Rng(1))
print("Q: orth err gpu", np.abs(qg.T @ qg - np.eye(25)).max())
print("Q: top-20 true-subspace capture  gpu %.3e  oracle %.3e" % (sinmax(qg, U[:, :20]), sinmax(qo, U[:, :20])))
print("Q: span(gpu) vs span(oracle) (all 25) %.3e" % sinmax(qo, qg))
f = eng.rsvd(At, cfg)
ug = f.U.cpu().numpy()
uo, so, vo = oracle.rsvd(A, 20, 5, 2, oracle.POWER, oracle.Rng(1))
print("U20: gpu vs oracle %.3e   gpu vs true %.3e   oracle vs true %.3e" % (
    sinmax(uo[:, :20], ug[:, :20]), sinmax(U[:, :20], ug[:, :20]), sinmax(U[:, :20], uo[:, :20])))
print("sigma gpu ", f.sigma.cpu().numpy()[18:25])
print("sigma orc ", so[18:25])
# stage-2 in numpy from the GPU Q
B = qg.T @ A
ub, sb, vbt = np.linalg.svd(B, full_matrices=False)
print("U20 from GPU Q + numpy SVD vs true %.3e" % sinmax(U[:, :20], (qg @ ub)[:, :20]))
