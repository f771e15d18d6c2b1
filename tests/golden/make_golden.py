"""Regenerate the golden Omega fixtures from the CPU oracle, whose normal
stream IS the reference's generator (std::mt19937_64 + std::normal_distribution
from the host libstdc++, sketch.hpp:19-59).  Run: python tests/golden/make_golden.py"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

CASES = [("omega_seed1_1024x25", 1024, 25, 1), ("omega_seed42_5x3", 5, 3, 42),
         ("omega_seed7_1000x4", 1000, 4, 7)]

if __name__ == "__main__":
    for name, n, l, seed in CASES:
        g = oracle.gaussian(n, l, oracle.Rng(seed))
        np.savez_compressed(os.path.join(HERE, name + ".npz"), omega=g, n=n, l=l, seed=seed)
        print(name, g.shape, g[0, 0])
