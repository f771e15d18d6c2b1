"""Edge cases of the hot path against the oracle / the reference's own unit
tests: exact-rank recovery in every mode (test_factor.cpp:24-35,
test_singlepass.cpp:25-35, 85-94; acceptance.cpp:180-212), the largest
admissible sketch l = min(m, n), the smallest (k = 1, p = 0), wide inputs,
strided / odd leading dimensions, non-finite inputs, single-pass shape
errors, and exact-rank inputs whose sketch is rank deficient (l > rank: the
padded-basis path of orthonormalize, core.hpp:93-95)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIG_TOL = 1e-10
ANG_TOL = 1e-8


def _t(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a)).cuda().t().contiguous().t()


def _np(x):
    return np.asfortranarray(x.cpu().numpy()) if hasattr(x, "cpu") else np.asarray(x)


def planted_rank(m, n, r, seed):
    """A rank-r matrix with O(1) singular values (tests/support/oracles.hpp style)."""
    rs = np.random.default_rng(seed)
    return np.asfortranarray(rs.standard_normal((m, r)) @ rs.standard_normal((r, n)))


def max_angle(x, y):
    r = y - x @ (x.T @ y)
    return float(np.arcsin(min(1.0, np.linalg.svd(r, compute_uv=False)[0]))) if x.size else 0.0


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("m,n,r,k,p", [(40, 30, 5, 5, 5), (300, 200, 7, 10, 6), (2000, 800, 12, 20, 12)])
def test_exact_rank_recovered_every_mode(eng, orc, mode, m, n, r, k, p):
    """test_factor.cpp:24-35 / acceptance.cpp:180-212: ||A - U S V^T|| <= 1e-10 ||A||
    with l > rank (rank-deficient sketch)."""
    a = planted_rank(m, n, r, 9)
    f = eng.rsvd(_t(a), eng.SketchConfig(k, p, 1, eng.RangeMode(mode), 3))
    u, s, v = _np(f.U), _np(f.sigma), _np(f.V)
    assert np.abs((u * s) @ v.T - a).max() <= 1e-10 * np.abs(a).max() * np.sqrt(m * n)
    assert np.abs(u.T @ u - np.eye(k + p)).max() < 1e-12  # padded to full width
    uo, so, vo = orc.rsvd(a, k, p, 1, mode, orc.Rng(3))
    assert np.max(np.abs(s[:r] - so[:r]) / so[:r]) < SIG_TOL
    assert max_angle(u[:, :r], uo[:, :r]) < ANG_TOL


def test_exact_rank_single_pass(eng, orc):
    """test_singlepass.cpp:25-35, 85-94: exact-rank recovery <= 1e-7."""
    rs = np.random.default_rng(6)
    q = np.linalg.qr(rs.standard_normal((30, 3)))[0]
    a_sym = np.asfortranarray((q * [3.0, -2.0, 1.0]) @ q.T)
    e = eng.spevd_hermitian(_t(a_sym), 3, 4, eng.Rng(6))
    u, lam = _np(e.U), _np(e.lam)
    assert np.abs((u * lam) @ u.T - a_sym).max() <= 1e-7 * np.abs(a_sym).max()
    a = planted_rank(25, 15, 4, 5)
    f = eng.spsvd_general(_t(a), 4, 3, eng.Rng(5))
    assert np.abs((_np(f.U) * _np(f.sigma)) @ _np(f.V).T - a).max() <= 1e-7 * np.abs(a).max()
    uo, so, vo = orc.spsvd_general(a, 4, 3, orc.Rng(5))
    assert np.max(np.abs(_np(f.sigma) - so) / so) < SIG_TOL


@pytest.mark.parametrize("m,n", [(300, 120), (120, 300), (64, 64)])
def test_largest_sketch_l_equals_min_dim(eng, orc, m, n):
    """k + p = min(m, n): the admissible maximum (rangefinder.hpp:52-54)."""
    rs = np.random.default_rng(m * n)
    a = np.asfortranarray(rs.standard_normal((m, n)))
    l = min(m, n)
    k = l - 4
    f = eng.rsvd(_t(a), eng.SketchConfig(k, 4, 0, eng.RangeMode.basic, 2))
    uo, so, vo = orc.rsvd(a, k, 4, 0, 0, orc.Rng(2))
    s = _np(f.sigma)
    assert np.max(np.abs(s - so) / so) < SIG_TOL
    # full-rank sketch: the factorization reproduces A
    assert np.abs((_np(f.U) * s) @ _np(f.V).T - a).max() < 1e-11 * np.abs(a).max() * l
    with pytest.raises(eng.DimensionError):
        eng.rsvd(_t(a), eng.SketchConfig(k, 5, 0, eng.RangeMode.basic, 2))


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_smallest_sketch_k1_p0(eng, orc, mode):
    rs = np.random.default_rng(1)
    u = np.linalg.qr(rs.standard_normal((500, 50)))[0]
    v = np.linalg.qr(rs.standard_normal((300, 50)))[0]
    a = np.asfortranarray((u * 0.5 ** np.arange(50)) @ v.T)
    f = eng.rsvd(_t(a), eng.SketchConfig(1, 0, 2, eng.RangeMode(mode), 4))
    uo, so, vo = orc.rsvd(a, 1, 0, 2, mode, orc.Rng(4))
    assert abs(_np(f.sigma)[0] - so[0]) / so[0] < SIG_TOL
    assert max_angle(_np(f.U), uo) < ANG_TOL


def test_wide_matrix_every_mode(eng, orc):
    rs = np.random.default_rng(2)
    u = np.linalg.qr(rs.standard_normal((300, 300)))[0]
    v = np.linalg.qr(rs.standard_normal((2000, 300)))[0]
    a = np.asfortranarray((u * 0.97 ** np.arange(300)) @ v.T)
    for mode, q in [(0, 0), (1, 2), (2, 1)]:
        f = eng.rsvd(_t(a), eng.SketchConfig(15, 5, q, eng.RangeMode(mode), 8))
        uo, so, vo = orc.rsvd(a, 15, 5, q, mode, orc.Rng(8))
        assert np.max(np.abs(_np(f.sigma)[:15] - so[:15]) / so[:15]) < SIG_TOL
        assert max_angle(_np(f.V)[:, :15], vo[:, :15]) < ANG_TOL


@pytest.mark.parametrize("ld_pad", [1, 3, 8])
def test_strided_leading_dimension(eng, orc, ld_pad):
    """A as a column-major view with ld > m (odd ld: the TMA path copies it
    once into an aligned workspace)."""
    import torch
    rs = np.random.default_rng(ld_pad)
    m, n = 333, 210
    a = np.asfortranarray(rs.standard_normal((m, n)) * 0.9 ** np.arange(n))
    big = torch.zeros((n, m + ld_pad), dtype=torch.float64, device="cuda")
    big[:, :m] = torch.from_numpy(np.ascontiguousarray(a.T))
    view = big.t()[:m, :]  # stride (1, m + ld_pad)
    f = eng.rsvd(view, eng.SketchConfig(10, 5, 1, eng.RangeMode.power, 5))
    uo, so, vo = orc.rsvd(a, 10, 5, 1, 1, orc.Rng(5))
    assert np.max(np.abs(_np(f.sigma)[:10] - so[:10]) / so[:10]) < SIG_TOL
    assert max_angle(_np(f.U)[:, :10], uo[:, :10]) < ANG_TOL


def test_non_finite_inputs_raise_numeric_error(eng):
    a = np.random.default_rng(0).standard_normal((100, 60))
    for bad in (np.nan, np.inf, -np.inf):
        b = a.copy()
        b[17, 23] = bad
        with pytest.raises(eng.NumericError):
            eng.rsvd(_t(b), eng.SketchConfig(5, 2, 1, eng.RangeMode.power, 1))
        with pytest.raises(eng.NumericError):
            eng.svd_small(_t(b))
        with pytest.raises(eng.NumericError):
            eng.spsvd_general(_t(b), 5, 2, eng.Rng(1))
    # the engine stays usable after the error
    f = eng.rsvd(_t(a), eng.SketchConfig(5, 2, 1, eng.RangeMode.power, 1))
    assert np.isfinite(_np(f.sigma)).all()


def test_single_pass_shape_errors(eng):
    a = _t(np.random.default_rng(0).standard_normal((30, 20)))
    with pytest.raises(eng.DimensionError):
        eng.spevd_hermitian(a, 3, 2, eng.Rng(1))  # not square
    sq = _t(np.eye(20))
    with pytest.raises(eng.DimensionError):
        eng.spevd_hermitian(sq, 18, 5, eng.Rng(1))  # k + p > n
    with pytest.raises(eng.ParameterError):
        eng.spevd_hermitian(sq, 0, 5, eng.Rng(1))
    with pytest.raises(eng.ParameterError):
        eng.spsvd_general(a, 3, -1, eng.Rng(1))
    with pytest.raises(eng.DimensionError):
        eng.spsvd_general(a, 18, 5, eng.Rng(1))


def test_rng_state_continues_after_device_calls(eng, orc):
    """sketch.hpp:19-45: the caller's Rng advances by exactly the draws consumed,
    through a whole factorization (Omega n x l), so host and device interleave."""
    a = planted_rank(200, 150, 20, 2)
    r_e, r_o = eng.Rng(77), orc.Rng(77)
    eng.rsvd(_t(a), eng.SketchConfig(8, 3, 1, eng.RangeMode.power, 0), r_e)
    orc.rsvd(a, 8, 3, 1, 1, r_o)
    x_e = [r_e.normal() for _ in range(5)]
    x_o = [r_o.normal() for _ in range(5)]
    assert np.allclose(x_e, x_o, rtol=1e-15, atol=0)


@pytest.mark.parametrize("l", [70, 150])
def test_joint_core_batched_block_jacobi(eng, orc, l):
    """l > 64: the two joint-core SVDs (G1, G2) run as one batched block-Jacobi
    launch; the result must equal the oracle's Kronecker route."""
    rs = np.random.default_rng(l)
    g1, h1, g2, h2 = (np.asfortranarray(rs.standard_normal((l, l))) for _ in range(4))
    c = eng.solve_joint_core(_t(g1), _t(h1), _t(g2), _t(h2))
    co = orc.solve_joint_core(g1, h1, g2, h2, route=1)
    assert np.abs(_np(c) - co).max() <= 1e-9 * np.abs(co).max()
