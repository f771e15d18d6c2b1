"""Warm-up factorizations, then exactly one more, of a BASELINE config on
cuda:0 (inputs from bench.make_input): the command ncu wraps for the
per-kernel launch lists and captures in profiles/.

  python tools/one_step.py C5 [warmup]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "C2"
    warm = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    cfg = bench.CONFIGS[config]
    a = bench.make_input(cfg, torch.device("cuda", 0))
    k, p, q = cfg["k"], cfg["p"], cfg["q"]

    def step():
        if cfg["alg"] == 5:
            return eng.spevd_hermitian(a, k, p, eng.Rng(bench.SEED_OMEGA))
        if cfg["alg"] == 6:
            return eng.spsvd_general(a, k, p, eng.Rng(bench.SEED_OMEGA))
        return eng.rsvd(a, eng.SketchConfig(k, p, q, eng.RangeMode[cfg["mode"]], bench.SEED_OMEGA))
    for _ in range(warm + 1):
        f = step()
    torch.cuda.synchronize()
    print(f"{config}: ok, sigma[0] = {float((f.sigma if hasattr(f, 'sigma') else f.lam)[0]):.15g}")


if __name__ == "__main__":
    main()
