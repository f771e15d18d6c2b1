import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2402_17794_b200 as eng, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_diag import lowrank_plus, _t
for (m, n, d) in [(1024, 512, 0.9), (300, 200, 0.5), (200, 130, 0.8)]:
    sig = np.r_[np.ones(10), 1e-4 * d ** np.arange(min(m, n) - 10)]
    a = lowrank_plus(m, n, sig, 0.0, 33)
    q = eng.orthonormalize(_t(a)).cpu().numpy()
    print(m, n, "Q orth dev", np.abs(q.T @ q - np.eye(n)).max(), flush=True)
    try:
        f = eng.svd_small(_t(a))
        u = f.U.cpu().numpy()
        print("ok U dev", np.abs(u.T @ u - np.eye(n)).max(), flush=True)
    except Exception as e:
        print("ERR", e, flush=True)
