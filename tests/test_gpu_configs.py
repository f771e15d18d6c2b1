"""Parity on the BASELINE configurations at full size (BASELINE.json configs
C1-C5; C5 holds its 68.7 GB A once in host RAM for the oracle, which runs
~30 s on the box's host cores).  Inputs are the bench's seeded synthetic
matrices (bench.make_input); the oracle runs on the box's host cores.

Tolerances (north_star): top-k singular values / |eigenvalues| within 1e-10
relative, canonical angles of the top-k subspaces <= 1e-8 rad.  The p
oversampled directions are round-off dominated in Alg 3 and
are not compared."""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SIG_TOL, ANG_TOL = 1e-10, 1e-8


def sin_max(x, y):
    r = y - x @ (x.T @ y)
    return float(np.linalg.svd(r, compute_uv=False)[0])


def _run(config):
    import torch
    import bench
    import oracle
    import paper_2402_17794_b200 as eng
    # "C5-dmma": C5 with the FP64 DMMA fused pass forced (the default for C5's
    # wide sketch is the sliced INT8 tensor-core pass, csrc/ozaki.cu)
    config, _, variant = config.partition("-")
    eng.set_ozaki_slices(0 if variant == "dmma" else -1)
    try:
        return _run_cfg(config, torch, bench, oracle, eng)
    finally:
        eng.set_ozaki_slices(-1)


def _run_cfg(config, torch, bench, oracle, eng):
    cfg = bench.CONFIGS[config]
    torch.cuda.set_device(0)
    a = bench.make_input(cfg, torch.device("cuda", 0))
    k, p, q = cfg["k"], cfg["p"], cfg["q"]
    if cfg["alg"] == 5:
        f = eng.spevd_hermitian(a, k, p, eng.Rng(bench.SEED_OMEGA))
        out = (f.U.cpu().numpy(), f.lam.cpu().numpy(), None)
    elif cfg["alg"] == 6:
        f = eng.spsvd_general(a, k, p, eng.Rng(bench.SEED_OMEGA))
        out = (f.U.cpu().numpy(), f.sigma.cpu().numpy(), f.V.cpu().numpy())
    else:
        mode = eng.RangeMode[cfg["mode"]]
        f = eng.rsvd(a, eng.SketchConfig(k, p, q, mode, bench.SEED_OMEGA))
        out = (f.U.cpu().numpy(), f.sigma.cpu().numpy(), f.V.cpu().numpy())
    torch.cuda.synchronize()
    a_host = np.asfortranarray(a.cpu().numpy())
    del a, f
    torch.cuda.empty_cache()
    oracle.set_threads(os.cpu_count() or 1)
    rng = oracle.Rng(bench.SEED_OMEGA)
    if cfg["alg"] == 5:
        ref = oracle.spevd_hermitian(a_host, k, p, rng)
        ref = (ref[0], ref[1], None)
    elif cfg["alg"] == 6:
        ref = oracle.spsvd_general(a_host, k, p, rng)
    else:
        mode = {"basic": 0, "power": 1, "power_ortho": 2}[cfg["mode"]]
        ref = oracle.rsvd(a_host, k, p, q, mode, rng)
    return cfg, out, ref


@pytest.mark.parametrize("config", ["C1", "C2", "C3", "C4", "C5", "C5-dmma"])
def test_config_parity(config):
    cfg, (u, s, v), (uo, so, vo) = _run(config)
    k = cfg["k"]
    print(f"{config}: sigma rel {np.max(np.abs(s[:k] - so[:k]) / np.abs(so[:k])):.3e}, "
          f"U angle {sin_max(u[:, :k], uo[:, :k]):.3e}")
    rel = np.max(np.abs(s[:k] - so[:k]) / np.abs(so[:k]))
    assert rel < SIG_TOL, f"{config}: top-k relative error {rel:.3e}"
    ang = sin_max(u[:, :k], uo[:, :k])
    orth = float(np.abs(u.T @ u - np.eye(u.shape[1])).max())
    orth_o = float(np.abs(uo.T @ uo - np.eye(uo.shape[1])).max())
    assert ang < ANG_TOL, f"{config}: U angle {ang:.3e} (orth gpu {orth:.1e}, oracle {orth_o:.1e})"
    if v is not None:
        assert sin_max(v[:, :k], vo[:, :k]) < ANG_TOL
