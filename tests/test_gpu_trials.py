"""Batched trials: the run_bounds / run_angles trial
loops (drivers.hpp:340-356, 400-431) with every pass over A shared by all
trials.  Each trial t must equal the single-trial call with Rng(seed + t) --
the oracle's and the engine's own -- to the parity tolerances (sigma 1e-10
relative, subspace angles 1e-8 rad); the residuals of run_bounds to the
spectral_norm tolerance."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a)).cuda().t().contiguous().t()


def haar(m, k, rs):
    q, r = np.linalg.qr(rs.standard_normal((m, k)))
    return q * np.sign(np.diag(r))


def make_matrix(m, n, seed, decay=0.9):
    rs = np.random.default_rng(seed)
    r = min(m, n)
    return np.asfortranarray((haar(m, r, rs) * decay ** np.arange(r)) @ haar(n, r, rs).T)


def max_angle(x, y):
    r = y - x @ (x.T @ y)
    return float(np.arcsin(min(1.0, np.linalg.svd(r, compute_uv=False)[0])))


MODES = [("basic", 0, 0), ("power", 1, 2), ("power_ortho", 2, 1)]


@pytest.mark.parametrize("mode_name,mode,q", MODES)
def test_range_basis_trials_match_single_trials(eng, orc, mode_name, mode, q):
    m, n, k, p, T, seed = 900, 500, 10, 5, 7, 40
    a = make_matrix(m, n, 1)
    cfg = eng.SketchConfig(k, p, q, eng.RangeMode[mode_name], seed)
    qs = eng.range_basis_trials(_t(a), cfg, T)
    assert len(qs) == T
    for t in range(T):
        qt = qs[t].cpu().numpy()
        assert np.abs(qt.T @ qt - np.eye(k + p)).max() < 1e-13
        qo = orc.range_basis(a, k, p, q, mode, orc.Rng(seed + t))
        assert max_angle(qo, qt) < 1e-8
        # the engine's own single-trial call: same subspace
        qs1 = eng.range_basis(_t(a), cfg, eng.Rng(seed + t)).cpu().numpy()
        assert max_angle(qs1, qt) < 1e-10


@pytest.mark.parametrize("mode_name,mode,q", MODES)
def test_rsvd_trials_match_oracle(eng, orc, mode_name, mode, q):
    m, n, k, p, T, seed = 1024, 700, 12, 8, 5, 3
    a = make_matrix(m, n, 2, 0.85)
    cfg = eng.SketchConfig(k, p, q, eng.RangeMode[mode_name], seed)
    fs = eng.rsvd_trials(_t(a), cfg, T)
    for t, f in enumerate(fs):
        uo, so, vo = orc.rsvd(a, k, p, q, mode, orc.Rng(seed + t))
        s = f.sigma.cpu().numpy()
        assert np.abs(s[:k] - so[:k]).max() <= 1e-10 * so[0]
        u, v = f.U.cpu().numpy(), f.V.cpu().numpy()
        assert max_angle(uo[:, :k], u[:, :k]) < 1e-8
        assert max_angle(vo[:, :k], v[:, :k]) < 1e-8
        # the factors are the engine's own single-trial factors (same sign
        # rule on U_B, core.hpp:115-122, applied per trial)
        f1 = eng.rsvd(_t(a), cfg, eng.Rng(seed + t))
        u1 = f1.U.cpu().numpy()
        assert np.abs(np.abs(np.sum(u1[:, :k] * u[:, :k], axis=0)) - 1).max() < 1e-9
        assert np.all(np.sum(u1[:, :k] * u[:, :k], axis=0) > 0)


def test_range_error_trials_match_oracle(eng, orc):
    """run_bounds (drivers.hpp:340-356): computed_range_error per trial; the
    bases are 600-wide, so the dense route is exact and the GPU matches the
    oracle to rounding."""
    m, n, k, p, q, T, seed = 800, 600, 8, 4, 1, 6, 11
    a = make_matrix(m, n, 3, 0.8)
    cfg = eng.SketchConfig(k, p, q, eng.RangeMode.power, seed)
    errs = eng.range_error_trials(_t(a), cfg, T)
    assert errs.shape == (T,)
    for t in range(T):
        qo = orc.range_basis(a, k, p, q, orc.POWER, orc.Rng(seed + t))
        eo = orc.computed_range_error(a, qo)
        assert abs(errs[t] - eo) <= 1e-8 * eo
        assert errs[t] >= 0.8 ** (k + p) * (1 - 1e-8)  # Eckart-Young floor


def test_trials_parameter_errors(eng):
    a = _t(make_matrix(60, 40, 4))
    with pytest.raises(eng.ParameterError):
        eng.range_basis_trials(a, eng.SketchConfig(3, 2, 0, eng.RangeMode.basic, 1), 0)
    with pytest.raises(eng.DimensionError):
        eng.rsvd_trials(a, eng.SketchConfig(40, 5, 0, eng.RangeMode.basic, 1), 2)
    with pytest.raises(eng.ParameterError):
        eng.range_error_trials(a, eng.SketchConfig(0, 2, 0, eng.RangeMode.basic, 1), 2)


def test_reconstruction_error_report(eng):
    """drivers.hpp:145-151 on the device vs numpy."""
    a = make_matrix(700, 550, 5, 0.95)
    f = eng.rsvd(_t(a), eng.SketchConfig(20, 5, 1, eng.RangeMode.power, 2))
    fro, spec = eng.reconstruction_error(_t(a), f)
    u, s, v = f.U.cpu().numpy(), f.sigma.cpu().numpy(), f.V.cpu().numpy()
    r = a - (u * s) @ v.T
    assert abs(fro - np.linalg.norm(r) / np.linalg.norm(a)) <= 1e-10 * fro
    assert abs(spec - np.linalg.norm(r, 2) / np.linalg.norm(a, 2)) <= 1e-9 * spec
