"""Full-size parity + timing of one BASELINE configuration: the engine on
cuda:0 against the CPU oracle on the box's host cores (same seeded input,
same Omega seed).  Writes gpurun_out/parity_<config>.json.  Intended for C5
(68.7 GB A, minutes of oracle time), which the pytest suite does not run.

  python tools/parity_config.py C5 [--no-oracle]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import oracle  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402


def sin_max(x, y):
    r = y - x @ (x.T @ y)
    return float(np.linalg.svd(r, compute_uv=False)[0])


def main():
    config = sys.argv[1]
    run_oracle = "--no-oracle" not in sys.argv
    cfg = bench.CONFIGS[config]
    k, p, q = cfg["k"], cfg["p"], cfg["q"]
    dev = torch.device("cuda", 0)
    t0 = time.time()
    a = bench.make_input(cfg, dev)
    torch.cuda.synchronize()
    t_gen = time.time() - t0

    def run():
        if cfg["alg"] == 5:
            return eng.spevd_hermitian(a, k, p, eng.Rng(bench.SEED_OMEGA))
        if cfg["alg"] == 6:
            return eng.spsvd_general(a, k, p, eng.Rng(bench.SEED_OMEGA))
        return eng.rsvd(a, eng.SketchConfig(k, p, q, eng.RangeMode[cfg["mode"]], bench.SEED_OMEGA))
    run()  # warm (grows the workspace arena)
    run()  # warm (the arena is merged into one allocation at this call)
    e = eng.default_engine()
    e.trace(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    f = run()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    trace = e.trace_report()
    e.trace(False)
    if cfg["alg"] == 5:
        u, s, v = f.U.cpu().numpy(), f.lam.cpu().numpy(), None
    else:
        u, s, v = f.U.cpu().numpy(), f.sigma.cpu().numpy(), f.V.cpu().numpy()
    out = {"config": config, "name": cfg["name"], "engine_ms": ms, "input_gen_s": t_gen,
           "trace_top": [(site, c, round(t, 3)) for site, c, t in trace[:12]]}
    if run_oracle:
        a_host = np.asfortranarray(a.cpu().numpy()) if a.stride(0) == 1 else a.t().cpu().numpy().T
        del a, f
        torch.cuda.empty_cache()
        oracle.set_threads(os.cpu_count() or 1)
        t0 = time.time()
        rng = oracle.Rng(bench.SEED_OMEGA)
        if cfg["alg"] == 5:
            uo, so = oracle.spevd_hermitian(a_host, k, p, rng)
            vo = None
        elif cfg["alg"] == 6:
            uo, so, vo = oracle.spsvd_general(a_host, k, p, rng)
        else:
            mode = {"basic": 0, "power": 1, "power_ortho": 2}[cfg["mode"]]
            uo, so, vo = oracle.rsvd(a_host, k, p, q, mode, rng)
        out["oracle_s"] = time.time() - t0
        out["oracle_threads"] = os.cpu_count()
        out["sigma_rel_err_topk"] = float(np.max(np.abs(s[:k] - so[:k]) / np.abs(so[:k])))
        out["angle_u_topk"] = float(np.arcsin(min(1.0, sin_max(u[:, :k], uo[:, :k]))))
        if v is not None:
            out["angle_v_topk"] = float(np.arcsin(min(1.0, sin_max(v[:, :k], vo[:, :k]))))
        out["pass"] = out["sigma_rel_err_topk"] < 1e-10 and out["angle_u_topk"] < 1e-8 and \
            out.get("angle_v_topk", 0.0) < 1e-8
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"parity_{config}.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
