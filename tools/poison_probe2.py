"""C1 then C2 rsvd in one process (as tests/test_gpu_configs.py runs them),
each checked against the oracle; optional RSVD_POISON."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import oracle  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402

oracle.set_threads(os.cpu_count() or 1)
order = sys.argv[1:] or ["C1", "C2"]
for c in order:
    cfg = bench.CONFIGS[c]
    a = bench.make_input(cfg, torch.device("cuda", 0))
    k, p, q = cfg["k"], cfg["p"], cfg["q"]
    mode = eng.RangeMode[cfg["mode"]]
    try:
        f = eng.rsvd(a, eng.SketchConfig(k, p, q, mode, bench.SEED_OMEGA))
    except Exception as e:  # noqa: BLE001
        print(c, "EXC", str(e)[:160], flush=True)
        continue
    u = f.U.cpu().numpy()
    ah = np.asfortranarray(a.cpu().numpy())
    uo, so, vo = oracle.rsvd(ah, k, p, q, {"basic": 0, "power": 1, "power_ortho": 2}[cfg["mode"]],
                             oracle.Rng(bench.SEED_OMEGA))
    r = u[:, :k] - uo[:, :k] @ (uo[:, :k].T @ u[:, :k])
    print(c, "angle %.2e orth %.1e sig %.2e" % (np.linalg.svd(r, compute_uv=False)[0],
          np.abs(u.T @ u - np.eye(u.shape[1])).max(),
          np.abs(f.sigma.cpu().numpy()[:k] - so[:k]).max()), "hw", flush=True)
