"""Time Alg 6's fused pass (fused.cu) against the two separate passes on a
C5-shaped problem (A 262144 x 32768 fp64, l = 550) with CUDA events.

  python tools/fused_bench.py [m n l] [--mb 1024,2048,4096] [--reps 3]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17794_b200 as eng  # noqa: E402

FP64 = 37.0e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dims", nargs="*", type=int, default=[262144, 32768, 550])
    ap.add_argument("--mb", default="2048")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--separate", action="store_true")
    a_ = ap.parse_args()
    m, n, l = a_.dims
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    a = torch.randn((n, m), dtype=torch.float64, device=dev, generator=g).t()
    oc = torch.randn((l, n), dtype=torch.float64, device=dev, generator=g).t()
    psi = torch.randn((l, m), dtype=torch.float64, device=dev, generator=g).t()
    out = {"m": m, "n": n, "l": l}

    def timeit(fn):
        fn()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(a_.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    for mb in [int(x) for x in a_.mb.split(",")]:
        ms = timeit(lambda: eng.debug_dual_pass(a, oc, psi, macroblock=mb))
        out[f"fused_mb{mb}_ms"] = ms
        out[f"fused_mb{mb}_frac_fp64"] = 4.0 * m * n * l / (ms * 1e-3) / FP64
    if a_.separate:
        ms1 = timeit(lambda: eng.apply(a, oc))
        ms2 = timeit(lambda: eng.apply_adjoint(a, psi))
        out["apply_ms"], out["adjoint_ms"] = ms1, ms2
        out["separate_frac_fp64"] = 4.0 * m * n * l / ((ms1 + ms2) * 1e-3) / FP64
    print(json.dumps(out))


if __name__ == "__main__":
    main()
