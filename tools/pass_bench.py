"""Time the streaming-pass kernels alone (live CUDA events inside the engine,
see rsvd_profile_enable) at BASELINE shapes; prints per-launch time and the
fraction of the FP64 / HBM roofline.  Usage: python tools/pass_bench.py [C2|C3|...] [reps]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17794_b200 as eng  # noqa: E402

SHAPES = {"C1": (2048, 1024, 25), "C2": (8192, 8192, 25), "C3": (65536, 16384, 110),
          "C4": (32768, 32768, 220), "C5s": (32768, 32768, 550)}
FP64, HBM = 37.0, 6550.7


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "C2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    m, n, l = SHAPES[which]
    torch.manual_seed(0)
    a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()  # column-major m x n
    x = torch.randn(l, n, dtype=torch.float64, device="cuda").t()
    y = torch.randn(l, m, dtype=torch.float64, device="cuda").t()
    e = eng.default_engine()
    out = {}
    for name, fn in (("apply", lambda: eng.apply(a, x)), ("adjoint", lambda: eng.apply_adjoint(a, y))):
        for _ in range(3):
            fn()
        e.profile(True)
        for _ in range(reps):
            fn()
        p = e.profile_read()[name]
        e.profile(False)
        ms = p["ms"] / p["launches"]
        fl, by = p["flops"] / p["launches"], p["bytes"] / p["launches"]
        roof = max(fl / (FP64 * 1e12), by / (HBM * 1e9))
        out[name] = {"shape": [m, n, l], "us": ms * 1e3, "tflops": fl / ms / 1e9,
                     "gbs": by / ms / 1e6, "frac_roofline": roof / (ms * 1e-3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
