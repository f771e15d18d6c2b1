"""Block-Jacobi sweep counts / times on l x l cores shaped like C3-C5
(RSVD_PROBE_FQ=1): svd_small of a matrix with the config's spectrum."""
import os
import sys

os.environ["RSVD_PROBE_FQ"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17794_b200 as eng  # noqa: E402

rs = np.random.default_rng(0)
for name, l, sig in [("C3", 110, np.exp(-np.arange(1, 111) / 50)),
                     ("C4", 220, np.arange(1, 221) ** -1.5 + 0.5),
                     ("C5", 550, np.exp(-np.arange(1, 551) / 200))]:
    u = np.linalg.qr(rs.standard_normal((l, l)))[0]
    v = np.linalg.qr(rs.standard_normal((l, l)))[0]
    a = torch.from_numpy(np.asfortranarray((u * sig) @ v.T)).cuda().t().contiguous().t()
    for _ in range(2):
        eng.svd_small(a)
    torch.cuda.synchronize()
