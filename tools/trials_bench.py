"""Batched trials vs the reference's per-trial loop on the GPU: T rsvd
factorizations with seeds seed..seed+T-1 as one rsvd_trials call (every pass
over A shared) against T single rsvd calls.  Usage:
python tools/trials_bench.py [C1|C2] [T]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "C1"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    cfg = bench.CONFIGS[config]
    a = bench.make_input(cfg, torch.device("cuda", 0))
    sk = eng.SketchConfig(cfg["k"], cfg["p"], cfg["q"], eng.RangeMode[cfg["mode"]], 1)

    def loop():
        return [eng.rsvd(a, sk, eng.Rng(1 + t)) for t in range(T)]

    def batched():
        return eng.rsvd_trials(a, sk, T)

    out = {"config": config, "trials": T}
    for name, fn in (("loop", loop), ("batched", batched)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        out[name + "_ms"] = (time.perf_counter() - t0) * 1e3 / reps
    out["speedup"] = out["loop_ms"] / out["batched_ms"]
    out["trials_per_s_batched"] = T * 1e3 / out["batched_ms"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
