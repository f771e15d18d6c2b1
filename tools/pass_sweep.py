"""Kernel-variant sweep for the l = 25 pass kernels (RSVD_PASS25_NN/TN):
time (live CUDA events) and check each against cuBLAS.  Usage:
python tools/pass_sweep.py C2 <variant>"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17794_b200 as eng  # noqa: E402
from tools.pass_bench import SHAPES, FP64, HBM  # noqa: E402


def main():
    which, reps = sys.argv[1], 30
    m, n, l = SHAPES[which]
    torch.manual_seed(0)
    a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    x = torch.randn(l, n, dtype=torch.float64, device="cuda").t()
    y = torch.randn(l, m, dtype=torch.float64, device="cuda").t()
    flush = torch.ones(1 << 27, dtype=torch.float32, device="cuda")
    e = eng.default_engine()
    out = {"variant": os.environ.get("RSVD_PASS25_NN", "0")}
    for name, fn, ref in (("apply", lambda: eng.apply(a, x), lambda: a @ x),
                          ("adjoint", lambda: eng.apply_adjoint(a, y), lambda: a.t() @ y)):
        r = fn()
        err = float((r - ref()).abs().max() / ref().abs().max())
        for _ in range(3):
            fn()
        e.profile(True)
        for i in range(reps):
            if m * n * 8 < (256 << 20) and not os.environ.get("NOFLUSH"):
                flush.sum()
            fn()
        p = e.profile_read()[name]
        e.profile(False)
        ms = p["ms"] / p["launches"]
        fl, by = p["flops"] / p["launches"], p["bytes"] / p["launches"]
        roof = max(fl / (FP64 * 1e12), by / (HBM * 1e9))
        out[name] = {"us": round(ms * 1e3, 2), "frac": round(roof / (ms * 1e-3), 4), "err": err}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
