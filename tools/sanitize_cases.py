"""Small cases of every synchronization-heavy kernel, for compute-sanitizer
(racecheck / synccheck; one tool per run): the TMA/mbarrier pass kernels
(split-K and stream-K), the fused Alg-6 pass (mbarrier ring + item ring +
tile semaphores), the cooperative CholeskyQR (l <= 32), the blocked
Cholesky, the cluster block-Jacobi (DSMEM), the exact-mode RNG patch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17794_b200 as eng  # noqa: E402


def t(a):
    return torch.from_numpy(np.asfortranarray(a)).cuda().t().contiguous().t()


def main():
    rs = np.random.default_rng(0)
    a = t(rs.standard_normal((700, 500)))
    y, w = eng.debug_dual_pass(a, t(rs.standard_normal((500, 60))), t(rs.standard_normal((700, 60))),
                               macroblock=128)
    f = eng.rsvd(a, eng.SketchConfig(10, 5, 1, eng.RangeMode.power, 1))          # l = 15: fused CholeskyQR
    f = eng.rsvd(t(rs.standard_normal((2000, 300))), eng.SketchConfig(60, 10, 1, eng.RangeMode.power_ortho, 2))
    s = eng.svd_small(t(rs.standard_normal((130, 130))))                       # block Jacobi, clusters
    g = eng.gaussian(3000, 7, eng.Rng(5))                                        # exact-mode patch
    torch.cuda.synchronize()
    print("sanitize cases ok", float(f.sigma[0]), float(s.sigma[0]), float(g[0, 0]), float(y[0, 0]))


if __name__ == "__main__":
    main()
