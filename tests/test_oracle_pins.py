"""Pin the CPU oracle (oracle/rsvd_oracle.cpp) to the reference before
trusting it as the parity checker.  The reference ships no golden vectors
(SURVEY.md §8c); these are its own unit-test properties and known answers,
ported from /root/reference/proj/tests/unit/test_{sketch,core,rangefinder,
factor,singlepass}.cpp (file:line in each docstring), plus the C++ standard's
mt19937_64 known answer and the committed golden Omega fixtures.  CPU only."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def random_matrix(orc, rows, cols, seed):
    """tests/support/oracles.hpp:56-64: same stream as rsvd::gaussian."""
    return orc.gaussian(rows, cols, orc.Rng(seed))


def planted_rank(orc, rows, cols, rank, seed):
    """tests/support/oracles.hpp:67-72."""
    f = random_matrix(orc, rows, rank, seed)
    g = random_matrix(orc, cols, rank, seed + 1)
    return f @ g.T


def spectral_norm(m):
    return np.linalg.norm(m, 2) if m.size else 0.0


def max_sine(x, y):
    """test_core.cpp:12-15."""
    r = y - x @ (x.T @ y)
    return np.linalg.svd(r, compute_uv=False)[0]


# ----------------------------------------------------------------- sketch
def test_mt19937_64_known_answer(orc):
    """C++ [rand.predef]: the 10000th output of default-seeded mt19937_64."""
    r = orc.Rng(5489)
    for _ in range(9999):
        r.raw()
    assert r.raw() == 9981545732273789042


def test_gaussian_reproducible_per_seed(orc):
    """test_sketch.cpp:11-20."""
    a = orc.gaussian(5, 3, orc.Rng(42))
    b = orc.gaussian(5, 3, orc.Rng(42))
    c = orc.gaussian(5, 3, orc.Rng(43))
    assert np.array_equal(a, b)
    assert np.abs(a - c).max() > 0


def test_gaussian_moments(orc):
    """test_sketch.cpp:22-29."""
    m = orc.gaussian(1000, 100, orc.Rng(7))
    assert abs(m.mean()) < 0.02
    assert abs(m.var(ddof=1) - 1.0) < 0.02


def test_gaussian_degenerate_and_rejects(orc):
    """test_sketch.cpp:31-35; sketch.hpp:49-51."""
    assert np.isfinite(orc.gaussian(1, 1, orc.Rng(1))[0, 0])
    with pytest.raises(orc.ParameterError):
        orc.gaussian(0, 1, orc.Rng(1))


def test_adjacent_seeds_uncorrelated(orc):
    """test_sketch.cpp:37-50."""
    ra, rb = orc.Rng(1000), orc.Rng(1001)
    a = np.array([ra.normal() for _ in range(100000)])
    b = np.array([rb.normal() for _ in range(100000)])
    assert abs(np.corrcoef(a, b)[0, 1]) <= 0.02


def test_gaussian_is_column_major_normal_stream(orc):
    """sketch.hpp:53-57: j outer, i inner; consecutive normal() calls."""
    r1, r2 = orc.Rng(9), orc.Rng(9)
    g = orc.gaussian(4, 3, r1)
    seq = np.array([r2.normal() for _ in range(12)])
    assert np.array_equal(g.ravel(order="F"), seq)


@pytest.mark.parametrize("name", ["omega_seed1_1024x25", "omega_seed42_5x3", "omega_seed7_1000x4"])
def test_golden_omega_fixtures(orc, name):
    """Committed fixtures (tests/golden/make_golden.py) of the libstdc++ stream."""
    d = np.load(os.path.join(GOLD, name + ".npz"))
    g = orc.gaussian(int(d["n"]), int(d["l"]), orc.Rng(int(d["seed"])))
    assert np.array_equal(g, d["omega"])


def test_rng_state_roundtrip(orc):
    r = orc.Rng(11)
    for _ in range(3):
        r.normal()
    st = r.get_state()
    x = [r.normal() for _ in range(5)]
    r2 = orc.Rng(0)
    r2.set_state(st)
    assert [r2.normal() for _ in range(5)] == x


# ------------------------------------------------------------------- core
def test_orthonormalize_known_answers(orc):
    """test_core.cpp:19-36."""
    q = orc.orthonormalize(np.eye(3))
    assert np.allclose(np.abs(np.diag(q.T @ np.eye(3))), 1, atol=1e-12)
    q = orc.orthonormalize(np.array([[3.0], [0.0], [4.0]]))
    sign = 1.0 if q[0, 0] > 0 else -1.0
    assert np.max(np.abs(sign * q[:, 0] - [0.6, 0.0, 0.8])) < 1e-12


def test_orthonormalize_span_pad_idempotent(orc):
    """test_core.cpp:38-67."""
    m = random_matrix(orc, 6, 3, 17)
    q = orc.orthonormalize(m)
    assert np.max(np.abs(q.T @ q - np.eye(3))) < 1e-12
    assert np.max(np.abs(m - q @ (q.T @ m))) < 1e-10 * np.abs(m).max()
    c = random_matrix(orc, 5, 1, 3)
    m = np.hstack([c, 2 * c, -0.5 * c])
    q = orc.orthonormalize(m)
    assert q.shape == (5, 3) and np.max(np.abs(q.T @ q - np.eye(3))) < 1e-12
    for seed in (1, 2, 3):
        m = random_matrix(orc, 10, 4, seed)
        q1 = orc.orthonormalize(m)
        assert max_sine(q1, orc.orthonormalize(q1)) < 1e-10


def test_orthonormalize_rejects(orc):
    """test_core.cpp:69-74."""
    with pytest.raises(orc.DimensionError):
        orc.orthonormalize(np.ones((2, 4)))
    bad = np.ones((3, 2))
    bad[1, 1] = np.nan
    with pytest.raises(orc.NumericError):
        orc.orthonormalize(bad)


def test_svd_small_known_answers_and_sign_rule(orc):
    """test_core.cpp:76-117."""
    _, s, _ = orc.svd_small(np.diag([3.0, 2.0, 1.0]))
    assert np.allclose(s, [3, 2, 1], atol=1e-12, rtol=0)
    _, s, _ = orc.svd_small(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert np.allclose(s, [1, 1], atol=1e-12, rtol=0)
    m = random_matrix(orc, 8, 5, 23)
    u, s, v = orc.svd_small(m)
    assert spectral_norm(m - (u * s) @ v.T) <= 1e-10 * (1 + spectral_norm(m))
    m = random_matrix(orc, 7, 4, 41)
    u1, _, v1 = orc.svd_small(m)
    u2, _, v2 = orc.svd_small(m)
    assert np.array_equal(u1, u2) and np.array_equal(v1, v2)
    for j in range(u1.shape[1]):
        assert u1[np.argmax(np.abs(u1[:, j])), j] >= 0


def test_evd_symmetric_known_answers(orc):
    """test_core.cpp:138-175."""
    _, lam = orc.evd_symmetric(np.diag([5.0, -2.0]))
    assert np.allclose(lam, [5, -2], atol=1e-12, rtol=0)
    u, lam = orc.evd_symmetric(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert np.allclose(lam, [1, -1], atol=1e-12, rtol=0)
    assert np.allclose(np.abs(u), 1 / np.sqrt(2), atol=1e-12)
    g = random_matrix(orc, 6, 6, 11)
    c = 0.5 * (g + g.T)
    u, lam = orc.evd_symmetric(c)
    assert spectral_norm(c - (u * lam) @ u.T) <= 1e-10 * (1 + spectral_norm(c))
    assert np.all(np.abs(lam[:-1]) >= np.abs(lam[1:]))
    with pytest.raises(orc.NumericError):
        orc.evd_symmetric(np.array([[1.0, 0.5], [-0.5, 1.0]]))


def test_solve_ls_properties(orc):
    """test_core.cpp:177-209."""
    h = random_matrix(orc, 3, 2, 5)
    assert np.max(np.abs(orc.solve_ls(np.eye(3), h) - h)) < 1e-13
    assert abs(orc.solve_ls(np.array([[1.0], [1.0]]), np.array([[1.0], [3.0]]))[0, 0] - 2) < 1e-12
    for seed in (1, 2, 3, 4):
        g = random_matrix(orc, 10, 4, seed)
        x0 = random_matrix(orc, 4, 3, seed + 100)
        assert np.max(np.abs(orc.solve_ls(g, g @ x0) - x0)) < 1e-9
    g = np.hstack([random_matrix(orc, 6, 2, 9), np.zeros((6, 1))])
    g[:, 2] = g[:, 0]
    h = random_matrix(orc, 6, 2, 10)
    x = orc.solve_ls(g, h)
    assert np.max(np.abs(g.T @ (g @ x - h))) < 1e-8


# ------------------------------------------------------------ rangefinder
def test_range_finders_capture_exact_rank(orc):
    """test_rangefinder.cpp:20-36, 74-80."""
    a = planted_rank(orc, 20, 10, 3, 4)
    nrm = spectral_norm(a)
    for seed in (1, 2, 3, 4, 5):
        q = orc.range_basis(a, 3, 2, 0, orc.BASIC, orc.Rng(seed))
        assert spectral_norm(a - q @ (q.T @ a)) <= 1e-10 * nrm
    a = planted_rank(orc, 20, 10, 3, 12)
    q = orc.range_basis(a, 3, 2, 2, orc.POWER_ORTHO, orc.Rng(3))
    assert spectral_norm(a - q @ (q.T @ a)) <= 1e-10 * spectral_norm(a)


def test_range_finders_reject(orc):
    """test_rangefinder.cpp:38-46."""
    a = np.eye(6, 4)
    with pytest.raises(orc.DimensionError):
        orc.range_basis(a, 4, 1, 0, orc.BASIC, orc.Rng(1))
    with pytest.raises(orc.DimensionError):
        orc.range_basis(a, 3, 2, 1, orc.POWER, orc.Rng(1))
    with pytest.raises(orc.ParameterError):
        orc.range_basis(a, 0, 2, 1, orc.POWER, orc.Rng(1))
    with pytest.raises(orc.ParameterError):
        orc.range_basis(a, 2, 1, -1, orc.POWER, orc.Rng(1))


def test_q0_collapses_variants_bitwise(orc):
    """test_rangefinder.cpp:48-56."""
    a = random_matrix(orc, 30, 12, 8)
    qb = orc.range_basis(a, 4, 3, 0, orc.BASIC, orc.Rng(5))
    qp = orc.range_basis(a, 4, 3, 0, orc.POWER, orc.Rng(5))
    qo = orc.range_basis(a, 4, 3, 0, orc.POWER_ORTHO, orc.Rng(5))
    assert np.array_equal(qb, qp) and np.array_equal(qb, qo)


def test_power_step_sketches_aat_a(orc):
    """test_rangefinder.cpp:58-72."""
    a = np.diag([2.0, 1.0, 0.5])
    a3 = (a @ a.T) @ a
    qp = orc.range_basis(a, 2, 1, 1, orc.POWER, orc.Rng(2))
    qd = orc.range_basis(a3, 2, 1, 0, orc.BASIC, orc.Rng(2))
    assert max_sine(qp, qd) < 1e-10


def test_range_error_respects_floor(orc):
    """test_rangefinder.cpp:113-130."""
    for mseed in (40, 41):
        a = random_matrix(orc, 60, 40, mseed)
        sv = np.linalg.svd(a, compute_uv=False)
        for seed in (1, 2, 3):
            for mode, q in ((orc.BASIC, 0), (orc.POWER, 1), (orc.POWER_ORTHO, 1)):
                qb = orc.range_basis(a, 6, 4, q, mode, orc.Rng(seed))
                assert spectral_norm(a - qb @ (qb.T @ a)) >= sv[10] - 1e-8 * sv[0]


# ----------------------------------------------------------------- factor
def test_rsvd_exact_recovery(orc):
    """test_factor.cpp:13-35."""
    u, s, v = orc.rsvd(np.diag([3.0, 2.0, 1.0]), 3, 0, 0, orc.BASIC, orc.Rng(1))
    assert np.allclose(s, [3, 2, 1], atol=1e-10, rtol=0)
    a = planted_rank(orc, 40, 30, 5, 9)
    nrm = spectral_norm(a)
    for mode in (orc.BASIC, orc.POWER, orc.POWER_ORTHO):
        for seed in (1, 2, 3):
            u, s, v = orc.rsvd(a, 5, 5, 1, mode, orc.Rng(seed))
            assert s.size == 10
            assert spectral_norm(a - (u * s) @ v.T) <= 1e-10 * nrm


def test_rsvd_basic_equals_power_q0(orc):
    """test_factor.cpp:73-83."""
    a = random_matrix(orc, 25, 18, 3)
    f1 = orc.rsvd(a, 5, 3, 7, orc.BASIC, orc.Rng(11))
    f2 = orc.rsvd(a, 5, 3, 0, orc.POWER, orc.Rng(11))
    for x, y in zip(f1, f2):
        assert np.array_equal(x, y)


def test_rsvd_factors_orthonormal(orc):
    """test_factor.cpp:46-60."""
    a = random_matrix(orc, 35, 25, 31)
    for mode in (orc.BASIC, orc.POWER, orc.POWER_ORTHO):
        u, s, v = orc.rsvd(a, 6, 4, 2, mode, orc.Rng(4))
        assert np.max(np.abs(u.T @ u - np.eye(10))) <= 1e-10
        assert np.max(np.abs(v.T @ v - np.eye(10))) <= 1e-10
        assert np.all(s[:-1] >= s[1:])


# ------------------------------------------------------------- singlepass
def test_spevd_properties(orc):
    """test_singlepass.cpp:15-54."""
    u, lam = orc.spevd_hermitian(np.eye(5), 3, 2, orc.Rng(1))
    assert np.allclose(lam, 1, atol=1e-8)
    h = random_matrix(orc, 30, 3, 6)
    d = np.array([(1.0 if i % 2 == 0 else -1.0) * (3 - i) for i in range(3)])
    a = (h * d) @ h.T
    a = 0.5 * (a + a.T)
    for seed in (1, 2, 3):
        u, lam = orc.spevd_hermitian(a, 3, 5, orc.Rng(seed))
        assert spectral_norm(a - (u * lam) @ u.T) <= 1e-7 * spectral_norm(a)
    g = random_matrix(orc, 40, 40, 8)
    cnt = {}
    orc.spevd_hermitian(0.5 * (g + g.T), 5, 3, orc.Rng(2), counters=cnt)
    assert cnt["apply"] == 1
    with pytest.raises(orc.DimensionError):
        orc.spevd_hermitian(random_matrix(orc, 6, 4, 1), 2, 1, orc.Rng(1))
    with pytest.raises(orc.NumericError):
        orc.spevd_hermitian(random_matrix(orc, 6, 6, 2), 2, 1, orc.Rng(1))


def test_spsvd_properties(orc):
    """test_singlepass.cpp:75-103."""
    _, s, _ = orc.spsvd_general(np.diag([3.0, 2.0, 1.0]), 3, 0, orc.Rng(4))
    assert np.allclose(s, [3, 2, 1], atol=1e-8, rtol=0)
    a = planted_rank(orc, 25, 15, 4, 5)
    for seed in (1, 2, 3):
        u, s, v = orc.spsvd_general(a, 4, 4, orc.Rng(seed))
        assert spectral_norm(a - (u * s) @ v.T) <= 1e-7 * spectral_norm(a)
    cnt = {}
    orc.spsvd_general(random_matrix(orc, 30, 20, 9), 4, 3, orc.Rng(3), counters=cnt)
    assert cnt == {"apply": 1, "adjoint": 1}


@pytest.mark.parametrize("l", [2, 6, 12, 20])
def test_joint_core_kronecker_equals_stacked(orc, l):
    """singlepass.hpp:84-101 vs the O(l^3) Kronecker route."""
    rs = np.random.default_rng(l)
    g1, h1, g2, h2 = (rs.standard_normal((l, l)) for _ in range(4))
    c0 = orc.solve_joint_core(g1, h1, g2, h2, route=0)
    c1 = orc.solve_joint_core(g1, h1, g2, h2, route=1)
    assert np.max(np.abs(c0 - c1)) <= 1e-12 * max(1.0, np.abs(c0).max()) * l


def test_joint_core_residual_vs_bruteforce(orc):
    """test_singlepass.cpp:105-143 (brute force by numpy lstsq)."""
    m, n, l = 20, 14, 6
    a = random_matrix(orc, m, n, 31)
    rng = orc.Rng(8)
    oc, orr = orc.gaussian(n, l, rng), orc.gaussian(m, l, rng)
    yc, yr = a @ oc, a.T @ orr
    qc, qr = orc.orthonormalize(yc), orc.orthonormalize(yr)
    g1, h1, g2, h2 = orr.T @ qc, yr.T @ qr, qr.T @ oc, qc.T @ yc
    c = orc.solve_joint_core(g1, h1, g2, h2, route=0)
    big = np.zeros((2 * l * l, l * l))
    rhs = np.zeros(2 * l * l)
    for col in range(l):
        big[col * l:(col + 1) * l, col * l:(col + 1) * l] = g1
        rhs[col * l:(col + 1) * l] = h1[:, col]
        for j in range(l):
            big[l * l + col * l + np.arange(l), j * l + np.arange(l)] = g2[j, col]
        rhs[l * l + col * l:l * l + (col + 1) * l] = h2[:, col]
    brute = np.linalg.lstsq(big, rhs, rcond=None)[0].reshape(l, l, order="F")

    def res(x):
        return np.sqrt(np.sum((g1 @ x - h1) ** 2) + np.sum((x @ g2 - h2) ** 2))
    assert res(c) <= res(brute) + 1e-9


# ------------------------------------------------- diagnostics (§8(f) rows 1, 3)
def test_oracle_spectral_norm_routes(orc):
    """core.hpp:188-221: dense route <= 512 equals sigma_max exactly; the power
    route converges to sigma_max (relative test 1e-10 between successive
    estimates) and is a lower bound."""
    rs = np.random.default_rng(0)
    a = rs.standard_normal((300, 200))
    assert abs(orc.spectral_norm(a) - np.linalg.norm(a, 2)) <= 1e-13 * np.linalg.norm(a, 2)
    u = np.linalg.qr(rs.standard_normal((700, 3)))[0]
    v = np.linalg.qr(rs.standard_normal((600, 3)))[0]
    b = (u * [5.0, 2.0, 1.0]) @ v.T
    s, it = orc.spectral_norm(b, with_iterations=True)
    assert it > 1 and abs(s - 5.0) <= 1e-12 * 5.0
    assert orc.spectral_norm(np.zeros((600, 600))) == 0.0


def test_oracle_range_error_and_sines(orc):
    """bounds.hpp:107-120 and angles.hpp:42-60 against numpy/scipy restatements."""
    import scipy.linalg as sl
    rs = np.random.default_rng(1)
    a = rs.standard_normal((120, 90))
    q = np.linalg.qr(rs.standard_normal((120, 10)))[0]
    assert abs(orc.computed_range_error(a, q) - np.linalg.norm(a - q @ (q.T @ a), 2)) < 1e-12
    with pytest.raises(orc.NumericError):
        orc.computed_range_error(a, 1.01 * q)
    x = np.linalg.qr(rs.standard_normal((80, 6)))[0]
    y = np.linalg.qr(x + 1e-2 * rs.standard_normal((80, 6)))[0]
    ref = np.sort(np.sin(sl.subspace_angles(x, y)))
    assert np.abs(orc.canonical_sines(x, y) - ref).max() < 1e-13
