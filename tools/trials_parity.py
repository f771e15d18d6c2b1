"""Parity of batched trials on a BASELINE configuration: every trial of one
rsvd_trials call (shared passes, INT8 tensor cores when T l is wide) against
the oracle's rsvd with the same seed.  Usage: python tools/trials_parity.py [C2] [T]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import oracle  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402


def sin_max(x, y):
    r = y - x @ (x.T @ y)
    return float(np.linalg.svd(r, compute_uv=False)[0])


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "C2"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cfg = bench.CONFIGS[config]
    a = bench.make_input(cfg, torch.device("cuda", 0))
    k, p, q = cfg["k"], cfg["p"], cfg["q"]
    sk = eng.SketchConfig(k, p, q, eng.RangeMode[cfg["mode"]], 1)
    fs = eng.rsvd_trials(a, sk, T)
    a_host = np.asfortranarray(a.cpu().numpy())
    oracle.set_threads(os.cpu_count() or 1)
    mode = {"basic": 0, "power": 1, "power_ortho": 2}[cfg["mode"]]
    worst = {"sigma": 0.0, "u": 0.0, "v": 0.0}
    for t in (0, T // 2, T - 1):
        uo, so, vo = oracle.rsvd(a_host, k, p, q, mode, oracle.Rng(1 + t))
        f = fs[t]
        s = f.sigma.cpu().numpy()
        worst["sigma"] = max(worst["sigma"], float(np.max(np.abs(s[:k] - so[:k]) / so[:k])))
        worst["u"] = max(worst["u"], sin_max(f.U.cpu().numpy()[:, :k], uo[:, :k]))
        worst["v"] = max(worst["v"], sin_max(f.V.cpu().numpy()[:, :k], vo[:, :k]))
    print(json.dumps({"config": config, "trials": T, **worst}))


if __name__ == "__main__":
    main()
