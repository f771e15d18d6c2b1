"""Where the end-to-end single-pass call (rsvd_spsvd_host / rsvd_spevd_host:
pinned host A streamed up in row panels into the pass) spends its time:
wall time per call, then one traced call (device time per launch site,
including the idle gap before each launch -- a fused-pass launch waiting for
its panel shows the upload).

  python tools/e2e_probe_sp.py C5|C4
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "C5"
    cfg = bench.CONFIGS[config]
    a = bench.make_input(cfg, torch.device("cuda", 0))
    m, n, k, p = cfg["m"], cfg["n"], cfg["k"], cfg["p"]
    pin = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
    pin.copy_(a.t())
    del a
    torch.cuda.empty_cache()
    a_host = pin.numpy().T
    u_h = torch.empty((k, m), dtype=torch.float64, pin_memory=True).numpy().T
    v_h = torch.empty((k, n), dtype=torch.float64, pin_memory=True).numpy().T
    s_h = torch.empty(k, dtype=torch.float64, pin_memory=True).numpy()
    out = (u_h, s_h, v_h) if cfg["alg"] == 6 else (u_h, s_h)
    fn = (lambda *x: eng.spsvd_host(*x, out=out)) if cfg["alg"] == 6 else (lambda *x: eng.spevd_host(*x, out=out))
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(a_host, k, p, eng.Rng(1))
        print(f"{config} host call {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    e = eng.default_engine()
    e.trace(True)
    t0 = time.perf_counter()
    fn(a_host, k, p, eng.Rng(1))
    print(f"traced call {1e3 * (time.perf_counter() - t0):.1f} ms")
    rows = e.trace_report()
    e.trace(False)
    tot = sum(r[2] for r in rows)
    print(f"device timeline {tot:.1f} ms")
    for site, cnt, ms in rows[:25]:
        print(f"  {site:28s} {cnt:4d} {ms:10.2f} ms")


if __name__ == "__main__":
    main()
