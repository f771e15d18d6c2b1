"""Accuracy and timing of the sliced INT8 tensor-core products (csrc/ozaki.cu).

  python tools/ozaki_check.py acc            # error vs a longdouble product, S = 4..8
  python tools/ozaki_check.py time [m n l]   # per-launch-site times of both products
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17794_b200 as eng  # noqa: E402


def colmajor(x):
    return torch.from_numpy(np.asfortranarray(x)).cuda().t().contiguous().t()


def acc():
    rs = np.random.default_rng(5)
    for (m, n, l) in [(300, 200, 25), (1000, 777, 110), (257, 4099, 220), (4100, 130, 30)]:
        a = rs.standard_normal((m, n)) * np.exp(rs.uniform(-3, 3, (m, 1)))
        for trans in (False, True):
            x = rs.standard_normal((m if trans else n, l))
            ref = (a.T.astype(np.longdouble) @ x.astype(np.longdouble)) if trans else (
                a.astype(np.longdouble) @ x.astype(np.longdouble))
            da, dx = colmajor(a), colmajor(x)
            t64 = (da.t() @ dx if trans else da @ dx).cpu().numpy()
            # normwise scale of each entry: |a| |x| (what a backward-stable product is measured against)
            sc = (np.abs(a).T @ np.abs(x)) if trans else (np.abs(a) @ np.abs(x))
            row = {"m": m, "n": n, "l": l, "trans": trans,
                   "fp64": float(np.max(np.abs(t64 - ref) / sc))}
            for s in (4, 5, 6, 7, 8):
                c = eng.debug_ozaki_gemm(da, dx, trans=trans, slices=s).cpu().numpy()
                row[f"S{s}"] = float(np.max(np.abs(c - ref) / sc))
            print(json.dumps(row), flush=True)


def timing(m, n, l):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    a = torch.randn((n, m), dtype=torch.float64, device=dev, generator=g).t()
    x = torch.randn((l, n), dtype=torch.float64, device=dev, generator=g).t()
    y = torch.randn((l, m), dtype=torch.float64, device=dev, generator=g).t()
    e = eng.default_engine()
    for s in (7, 6):
        for trans, v in ((False, x), (True, y)):
            eng.debug_ozaki_gemm(a, v, trans=trans, slices=s)
            torch.cuda.synchronize()
            e.trace(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            c = eng.debug_ozaki_gemm(a, v, trans=trans, slices=s)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            rep = e.trace_report()
            e.trace(False)
            ref = (a.t() @ v) if trans else (a @ v)
            err = float((c - ref).abs().max() / ref.abs().max())
            print(json.dumps({"S": s, "trans": trans, "m": m, "n": n, "l": l, "ms": ms,
                              "fp64_equiv_tflops": 2.0 * m * n * l / (ms * 1e-3) / 1e12,
                              "max_err_vs_torch": err}), flush=True)
            for r in rep:
                print("   ", r, flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "time":
        d = [int(v) for v in sys.argv[2:5]] or [32768, 32768, 550]
        timing(*d)
    else:
        acc()
