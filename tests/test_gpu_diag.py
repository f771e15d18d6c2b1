"""GPU parity of the residual / subspace diagnostics:
singular_values, spectral_norm (core.hpp:180-221), computed_range_error
(bounds.hpp:107-120), canonical_sines / subspace_quality (angles.hpp:42-78),
through the C ABI against the CPU oracle on the same seeded inputs.

Tolerances: dense singular values 1e-12 relative to sigma_max (both are
backward-stable SVDs of the same matrix); the power iteration follows the
reference's own iterates from the same LCG start vector, so the GPU estimate
matches the oracle's to 1e-9 relative (the stopping test is |est - sigma| <=
1e-10 est, so a one-step difference in where it stops moves the result by at
most ~1e-10); sines 1e-12 absolute (they are singular values of an
orthonormal-column residual, so absolute error is the right scale)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a)).cuda().t().contiguous().t()


def haar(m, k, rs):
    q, r = np.linalg.qr(rs.standard_normal((m, k)))
    return q * np.sign(np.diag(r))


def lowrank_plus(m, n, sig, noise, seed):
    rs = np.random.default_rng(seed)
    u, v = haar(m, len(sig), rs), haar(n, len(sig), rs)
    return np.asfortranarray((u * sig) @ v.T + noise * rs.standard_normal((m, n)))


@pytest.mark.parametrize("m,n", [(40, 30), (30, 40), (513, 200), (700, 520)])
def test_singular_values(eng, orc, m, n):
    a = np.asfortranarray(np.random.default_rng(m + n).standard_normal((m, n)))
    g, o = eng.singular_values(_t(a)).cpu().numpy(), orc.singular_values(a)
    assert np.abs(g - o).max() <= 1e-12 * o[0]
    # host-array path gives the same values
    assert np.abs(eng.singular_values(a) - o).max() <= 1e-12 * o[0]


@pytest.mark.parametrize("m,n,seed", [(600, 700, 0), (2048, 1024, 1), (1500, 3000, 2)])
def test_spectral_norm_power_route(eng, orc, m, n, seed):
    """min(m, n) > 512: the power iteration on M^T M (core.hpp:194-220)."""
    sig = np.r_[1.0, 0.9, 0.5 * np.ones(20)]
    a = lowrank_plus(m, n, sig, 1e-3, seed)
    o, it = orc.spectral_norm(a, with_iterations=True)
    assert it > 1
    g = eng.spectral_norm(_t(a))
    assert abs(g - o) <= 1e-9 * o
    assert abs(eng.spectral_norm(a) - o) <= 1e-9 * o


def test_spectral_norm_gaussian_slow_convergence(eng, orc):
    """A Gaussian matrix has a small top gap: hundreds of power steps."""
    a = np.asfortranarray(np.random.default_rng(0).standard_normal((600, 700)))
    o, it = orc.spectral_norm(a, with_iterations=True)
    assert it > 100
    assert abs(eng.spectral_norm(_t(a)) - o) <= 1e-9 * o


@pytest.mark.parametrize("m,n", [(100, 512), (512, 2000), (37, 5)])
def test_spectral_norm_dense_route(eng, orc, m, n):
    a = np.asfortranarray(np.random.default_rng(5).standard_normal((m, n)))
    o = orc.spectral_norm(a)
    assert abs(eng.spectral_norm(_t(a)) - o) <= 1e-12 * o


def test_spectral_norm_edge_cases(eng, orc):
    z = np.zeros((600, 600), order="F")
    assert eng.spectral_norm(_t(z)) == 0.0 == orc.spectral_norm(z)
    bad = np.ones((600, 600), order="F")
    bad[3, 4] = np.nan
    with pytest.raises(eng.NumericError):
        eng.spectral_norm(_t(bad))
    with pytest.raises(orc.NumericError):
        orc.spectral_norm(bad)


@pytest.mark.parametrize("m,n,k,p,q", [(2048, 1024, 20, 5, 0), (1024, 1536, 10, 5, 1),
                                       (300, 200, 8, 2, 0)])
def test_computed_range_error(eng, orc, m, n, k, p, q):
    sig = 10.0 ** (-np.arange(min(m, n)) / 40.0)
    a = lowrank_plus(m, n, sig, 0.0, 11)
    qb = orc.range_basis(a, k, p, q, orc.POWER if q else orc.BASIC, orc.Rng(3))
    o = orc.computed_range_error(a, qb)
    g = eng.computed_range_error(_t(a), _t(qb))
    tol = 1e-9 if min(m, n) > 512 else 1e-11
    assert abs(g - o) <= tol * o + 1e-15
    # Eckart-Young floor (reference test_rangefinder.cpp:113-130): >= sigma_{l+1}
    assert g >= sig[k + p] * (1 - 1e-8)


def test_computed_range_error_preconditions(eng):
    a = np.random.default_rng(0).standard_normal((50, 40))
    q = np.linalg.qr(np.random.default_rng(1).standard_normal((50, 5)))[0]
    with pytest.raises(eng.DimensionError):
        eng.computed_range_error(a, q[:49])
    with pytest.raises(eng.NumericError, match="not orthonormal"):
        eng.computed_range_error(a, 2.0 * q)


@pytest.mark.parametrize("m,kx,ky,eps", [(100, 5, 5, 1e-3), (2000, 25, 25, 1e-6), (500, 30, 20, 1e-2),
                                          (400, 70, 70, 1e-4)])
def test_canonical_sines(eng, orc, m, kx, ky, eps):
    rs = np.random.default_rng(m + kx)
    x = haar(m, kx, rs)
    y = np.linalg.qr(x[:, :ky] + eps * rs.standard_normal((m, ky)))[0]
    o = orc.canonical_sines(x, y)
    g = eng.canonical_sines(_t(x), _t(y)).cpu().numpy()
    assert g.shape == o.shape == (min(kx, ky),)
    assert np.all(np.diff(g) >= 0) and g.min() >= 0 and g.max() <= 1
    assert np.abs(g - o).max() <= 1e-12


def test_canonical_sines_identical_and_orthogonal(eng):
    rs = np.random.default_rng(3)
    x = haar(64, 8, rs)
    assert np.abs(eng.canonical_sines(x, x)).max() < 1e-14
    z = haar(64, 16, rs)
    s = eng.canonical_sines(z[:, :8], z[:, 8:])
    assert np.abs(s - 1.0).max() < 1e-14  # clamped to [0, 1]
    with pytest.raises(eng.NumericError, match="X: columns are not orthonormal"):
        eng.canonical_sines(3.0 * x, x)
    with pytest.raises(eng.DimensionError):
        eng.canonical_sines(x, x[:63])


def test_subspace_quality_of_rsvd(eng, orc):
    """angles.hpp:62-78 on a real factorization: GPU rsvd vs the oracle's
    exact SVD of A; sin_theta / sin_nu are tiny above the gap."""
    m, n, k = 1024, 512, 10
    sig = np.r_[np.ones(k), 1e-4 * 0.9 ** np.arange(n - k)]
    a = lowrank_plus(m, n, sig, 0.0, 21)
    res = eng.rsvd(_t(a), eng.SketchConfig(k, 5, 1, eng.RangeMode.power, 7))
    full = eng.svd_small(_t(a))
    rep = eng.subspace_quality(full, k, res)
    assert rep.k == k
    st, sn = rep.sin_theta.cpu().numpy(), rep.sin_nu.cpu().numpy()
    assert st.max() < 1e-6 and sn.max() < 1e-6
    # against the oracle's sines of the same pair of bases
    ou, _, ov = orc.svd_small(a)
    ru, rv = res.U.cpu().numpy(), res.V.cpu().numpy()
    assert np.abs(st - orc.canonical_sines(ou[:, :k], ru[:, :k])).max() < 1e-12
    assert np.abs(sn - orc.canonical_sines(ov[:, :k], rv[:, :k])).max() < 1e-12


@pytest.mark.parametrize("m,n,decay", [(1024, 512, 0.9), (300, 200, 0.5), (200, 130, 0.8)])
def test_svd_small_graded_rank_deficient_wide(eng, orc, m, n, decay):
    """l > 64 (block Jacobi) on a numerically rank-deficient, strongly graded
    matrix (singular values spanning > 1/u): the case the reference meets in
    subspace_quality(a, ...) and run_image (k up to 800).  Singular values to
    absolute accuracy u * sigma_max like the reference's BDCSVD, orthonormal
    factors, backward error ~u ||A||."""
    sig = np.r_[np.ones(10), 1e-4 * decay ** np.arange(min(m, n) - 10)]
    a = lowrank_plus(m, n, sig, 0.0, 33)
    f = eng.svd_small(_t(a))
    u, s, v = f.U.cpu().numpy(), f.sigma.cpu().numpy(), f.V.cpu().numpy()
    _, so, _ = orc.svd_small(a)
    assert np.abs(s - so).max() <= 1e-13 * so[0]
    r = min(m, n)
    assert np.abs(u.T @ u - np.eye(r)).max() < 1e-12
    assert np.abs(v.T @ v - np.eye(r)).max() < 1e-12
    assert np.abs((u * s) @ v.T - a).max() < 1e-13 * so[0]
