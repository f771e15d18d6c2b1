"""Live launch-site breakdown of one factorization (no profiler): every launch
site's device time including the idle gap before it.  Usage:
python tools/trace_step.py [C2|C1|C3|C4|C5] [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "C2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    cfg = bench.CONFIGS[config]
    a = bench.make_input(cfg, torch.device("cuda", 0))
    e = eng.default_engine()
    k, p, q = cfg["k"], cfg["p"], cfg["q"]

    def step():
        if cfg["alg"] == 5:
            return eng.spevd_hermitian(a, k, p, eng.Rng(1))
        if cfg["alg"] == 6:
            return eng.spsvd_general(a, k, p, eng.Rng(1))
        return eng.rsvd(a, eng.SketchConfig(k, p, q, eng.RangeMode[cfg["mode"]], 1))
    for _ in range(3):
        step()
    e.trace(True)
    for _ in range(steps):
        step()
    rows = e.trace_report()
    e.trace(False)
    tot = sum(r[2] for r in rows)
    print(f"{config}: {tot / steps:.3f} ms per factorization (device, incl. gaps)")
    for site, cnt, ms in rows:
        print(f"  {site:28s} {cnt // steps:4d}/step {1000 * ms / steps:9.1f} us/step {100 * ms / tot:5.1f}%")


if __name__ == "__main__":
    main()
