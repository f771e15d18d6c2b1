"""GPU parity tests: the CUDA engine (through the C ABI) against the CPU oracle
on the same seeded inputs.  Tolerances (BASELINE.json north_star): singular
values 1e-10 relative, canonical angles <= 1e-8 rad for the top-k triples; the
Omega / Psi stream bit-exact (exact mode: near-midpoint polar inputs take the
host glibc log, rng.cu)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIG_TOL = 1e-10
ANG_TOL = 1e-8


def _t(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a)).cuda().t().contiguous().t()


def _np(t):
    return np.asfortranarray(t.cpu().numpy()) if hasattr(t, "cpu") else np.asarray(t)


def max_angle(x, y):
    """Largest canonical angle between range(x) and range(y), both orthonormal
    with equal width, by the projection route of the reference's
    canonical_sines (angles.hpp:42-57): sin = sigma_max((I - X X^T) Y)."""
    if not x.size:
        return 0.0
    r = y - x @ (x.T @ y)
    s = np.linalg.svd(r, compute_uv=False)[0]
    return float(np.arcsin(min(1.0, s)))


def haar_test_matrix(m, n, sigma, seed):
    rs = np.random.default_rng(seed)
    u, r = np.linalg.qr(rs.standard_normal((m, len(sigma))))
    u *= np.sign(np.diag(r))
    v, r = np.linalg.qr(rs.standard_normal((n, len(sigma))))
    v *= np.sign(np.diag(r))
    return np.asfortranarray((u * sigma) @ v.T)


# ------------------------------------------------------------------ Omega
@pytest.mark.parametrize("n,l,seed", [(5, 3, 42), (1, 1, 1), (1000, 25, 7), (8192, 25, 1),
                                      (3, 7, 99), (4097, 11, 12345)])
def test_gaussian_stream_matches_libstdcxx(eng, orc, n, l, seed):
    r_g, r_o = eng.Rng(seed), orc.Rng(seed)
    g = eng.gaussian(n, l, r_g)
    o = orc.gaussian(n, l, r_o)
    assert_stream_equal(g, o)
    # the engine state advanced exactly like the host library's
    assert_state_equal(r_g, r_o)


def assert_stream_equal(g, o):
    diff = g != o
    assert not diff.any(), f"{int(diff.sum())} of {g.size} normals differ from libstdc++"
    # bitwise, not just ==: -0.0 vs 0.0 and the sign bits must match too
    assert np.array_equal(np.asarray(g).view(np.uint64), np.asarray(o).view(np.uint64))


def assert_state_equal(r_g, r_o):
    so = r_o.get_state()
    sg = r_g.state
    assert so.pos == sg.pos
    assert list(so.mt) == list(sg.mt)
    assert so.has_cached == sg.has_cached
    if so.has_cached:
        assert np.float64(so.cached).view(np.uint64) == np.float64(sg.cached).view(np.uint64)


@pytest.mark.parametrize("n,l,seed", [(100000, 25, 3), (333333, 7, 11)])
def test_gaussian_long_stream_jump_ahead(eng, orc, n, l, seed):
    """> 2 segments of 319488 draws: the segmented generator seeded by MT
    jump-ahead windows (rng.cu / mtjump.cpp) must reproduce the stream."""
    r_g, r_o = eng.Rng(seed), orc.Rng(seed)
    r_o.normal()  # leave a cached variate in both so the carry path is covered too
    r_g.normal()
    g = eng.gaussian(n, l, r_g)
    o = orc.gaussian(n, l, r_o)
    assert_stream_equal(g, o)
    assert_state_equal(r_g, r_o)


def test_gaussian_stream_after_mixed_lengths(eng, orc):
    """The jump tables are cached per handle and per segment length: streams of
    other lengths (and so other segment schedules) in between must not change
    a later stream (the C2 sketch 8192 x 25 seed 1 is checked before and after)."""
    def check(n, l, seed):
        r_g, r_o = eng.Rng(seed), orc.Rng(seed)
        g = eng.gaussian(n, l, r_g)
        o = orc.gaussian(n, l, r_o)
        assert_stream_equal(g, o)
        assert_state_equal(r_g, r_o)
    for n, l, seed in [(8192, 25, 1), (100000, 25, 3), (333333, 7, 11), (8192, 25, 1),
                       (4097, 11, 12345), (100000, 25, 3), (8192, 25, 1), (1000, 25, 7),
                       (8192, 25, 1)]:
        check(n, l, seed)


def test_gaussian_consecutive_calls_carry_cached_variate(eng, orc):
    """Alg 6 draws Omega_c then Psi from one Rng (singlepass.hpp:119-120)."""
    r_g, r_o = eng.Rng(8), orc.Rng(8)
    for (n, l) in [(7, 3), (5, 1), (9, 2), (1, 1), (333, 5)]:
        g = eng.gaussian(n, l, r_g)
        o = orc.gaussian(n, l, r_o)
        assert_stream_equal(g, o)
    assert_state_equal(r_g, r_o)


def test_gaussian_c5_omega_then_psi_exact(eng, orc):
    """C5's two test matrices from ONE Rng(1) (singlepass.hpp:119-120):
    Omega_c 32768 x 550 then Psi 262144 x 550 -- 1.62e8 normals, every one
    bit-identical to libstdc++'s normal_distribution over mt19937_64."""
    r_g, r_o = eng.Rng(1), orc.Rng(1)
    for (n, l) in [(32768, 550), (262144, 550)]:
        g = eng.gaussian(n, l, r_g)
        o = orc.gaussian(n, l, r_o)
        assert_stream_equal(g, o)
        del g, o
    assert_state_equal(r_g, r_o)


def test_gaussian_odd_counts_patch_the_cached_variate(eng, orc):
    """Odd-length streams end with a cached second variate; in exact mode a
    near-midpoint completing pair must patch the cache too.  Many short odd
    streams from one Rng exercise that (each hands its cache to the next)."""
    r_g, r_o = eng.Rng(2024), orc.Rng(2024)
    for t in range(60):
        n, l = 3 + 2 * (t % 7), 1 + 2 * (t % 3)
        assert_stream_equal(eng.gaussian(n, l, r_g), orc.gaussian(n, l, r_o))
        assert_state_equal(r_g, r_o)


def test_gaussian_rejects_degenerate_shape(eng):
    with pytest.raises(eng.ParameterError):
        eng.gaussian(0, 3, eng.Rng(1))


# ------------------------------------------------------------ pass engine
@pytest.mark.parametrize("m,n,l", [(2048, 1024, 25), (1000, 777, 25), (300, 5000, 40),
                                   (4096, 512, 110), (513, 129, 1), (64, 64, 64), (3, 3, 3),
                                   (5, 7, 2), (1025, 2049, 57)])
def test_apply_and_adjoint_match_fp64_gemm(eng, m, n, l):
    rs = np.random.default_rng(m * 7 + n)
    a = rs.standard_normal((m, n))
    x = rs.standard_normal((n, l))
    y = rs.standard_normal((m, l))
    ya = _np(eng.apply(_t(a), _t(x)))
    za = _np(eng.apply_adjoint(_t(a), _t(y)))
    ref_y, ref_z = a @ x, a.T @ y
    tol = 1e-13 * np.sqrt(max(n, m))
    assert np.max(np.abs(ya - ref_y)) <= tol * np.max(np.abs(ref_y)) + 1e-300
    assert np.max(np.abs(za - ref_z)) <= tol * np.max(np.abs(ref_z)) + 1e-300


def test_call_waits_for_inputs_queued_on_default_stream(eng):
    """The engine runs on its own non-blocking stream when the caller is on the
    legacy default stream: it must still wait for the caller's queued kernels
    that produce its inputs (here a ~30 ms cuBLAS product issued right before
    the call)."""
    import torch
    torch.cuda.synchronize()
    g = torch.Generator(device="cuda").manual_seed(5)
    b = torch.randn(6144, 6144, dtype=torch.float64, device="cuda", generator=g)
    x = torch.randn(25, 6144, dtype=torch.float64, device="cuda", generator=g).t()
    torch.cuda.synchronize()
    assert torch.cuda.current_stream().cuda_stream == 0
    a = b @ b  # asynchronous on the default stream
    y = eng.apply(a, x)
    ref = a @ x
    assert float((y - ref).abs().max() / ref.abs().max()) < 1e-13


def test_pass_is_bitwise_deterministic(eng):
    rs = np.random.default_rng(5)
    a, x = _t(rs.standard_normal((4096, 8192))), _t(rs.standard_normal((4096, 25)))
    z1 = _np(eng.apply_adjoint(a, x))
    z2 = _np(eng.apply_adjoint(a, x))
    assert np.array_equal(z1, z2)


# ----------------------------------------------------------- core kernels
@pytest.mark.parametrize("m,l", [(3, 1), (6, 3), (10, 4), (257, 25), (8192, 25), (3000, 64),
                                 (5000, 100), (700, 220)])
def test_orthonormalize_matches_householder_span(eng, orc, m, l):
    rs = np.random.default_rng(m + l)
    y = rs.standard_normal((m, l))
    q = _np(eng.orthonormalize(_t(y)))
    qo = orc.orthonormalize(y)
    assert np.max(np.abs(q.T @ q - np.eye(l))) < 1e-12
    assert max_angle(q, qo) < 1e-10
    assert np.max(np.abs(y - q @ (q.T @ y))) < 1e-10 * np.max(np.abs(y))


@pytest.mark.parametrize("m,l,cond", [(4000, 110, 1e12), (3000, 220, 1e10), (6000, 550, 1e6),
                                      (2000, 40, 1e14)])
def test_orthonormalize_ill_conditioned_wide(eng, orc, m, l, cond):
    """Blocked multi-CTA CholeskyQR (l > 32) incl. the shifted restart: an
    ill-conditioned Y (graded singular values down to 1/cond) must come out
    orthonormal and spanning Y."""
    rs = np.random.default_rng(l)
    u, _ = np.linalg.qr(rs.standard_normal((m, l)))
    v, _ = np.linalg.qr(rs.standard_normal((l, l)))
    y = np.asfortranarray((u * np.logspace(0, -np.log10(cond), l)) @ v)
    q = _np(eng.orthonormalize(_t(y)))
    assert np.max(np.abs(q.T @ q - np.eye(l))) < 1e-12
    assert np.max(np.abs(y - q @ (q.T @ y))) < 1e-10 * np.max(np.abs(y))


def test_orthonormalize_pads_rank_deficient(eng):
    rs = np.random.default_rng(3)
    c = rs.standard_normal((5, 1))
    m = np.hstack([c, 2 * c, -0.5 * c])
    q = _np(eng.orthonormalize(_t(m)))
    assert q.shape == (5, 3)
    assert np.max(np.abs(q.T @ q - np.eye(3))) < 1e-12
    assert np.max(np.abs(m - q @ (q.T @ m))) < 1e-10 * np.max(np.abs(m))


def test_orthonormalize_rejects(eng):
    with pytest.raises(eng.DimensionError):
        eng.orthonormalize(_t(np.ones((2, 4))))
    bad = np.ones((3, 2))
    bad[1, 1] = np.nan
    with pytest.raises(eng.NumericError):
        eng.orthonormalize(_t(bad))


@pytest.mark.parametrize("m,n", [(3, 3), (2, 2), (8, 5), (7, 4), (5, 8), (25, 1024), (110, 110),
                                 (40, 40)])
def test_svd_small_matches_oracle(eng, orc, m, n):
    rs = np.random.default_rng(m * 100 + n)
    a = rs.standard_normal((m, n))
    f = eng.svd_small(_t(a))
    u, s, v = _np(f.U), _np(f.sigma), _np(f.V)
    uo, so, vo = orc.svd_small(a)
    assert np.max(np.abs(s - so) / so) < 1e-12
    # sign rule makes factors comparable, not just products
    assert np.max(np.abs(u - uo)) < 1e-9
    assert np.max(np.abs(v - vo)) < 1e-9
    r = min(m, n)
    assert np.max(np.abs(u.T @ u - np.eye(r))) < 1e-10
    assert np.max(np.abs(v.T @ v - np.eye(r))) < 1e-10


def test_svd_small_known_answers(eng):
    f = eng.svd_small(_t(np.diag([3.0, 2.0, 1.0])))
    assert np.allclose(_np(f.sigma), [3, 2, 1], atol=1e-12, rtol=0)
    f = eng.svd_small(_t(np.array([[0.0, 1.0], [1.0, 0.0]])))
    assert np.allclose(_np(f.sigma), [1, 1], atol=1e-12, rtol=0)


@pytest.mark.parametrize("n", [2, 6, 30, 110, 220])
def test_evd_symmetric_matches_oracle(eng, orc, n):
    rs = np.random.default_rng(n)
    g = rs.standard_normal((n, n))
    c = 0.5 * (g + g.T)
    e = eng.evd_symmetric(_t(c))
    u, lam = _np(e.U), _np(e.lam)
    uo, lo = orc.evd_symmetric(c)
    assert np.max(np.abs(lam - lo)) < 1e-12 * np.max(np.abs(lo))
    assert np.all(np.abs(lam[:-1]) >= np.abs(lam[1:]))
    assert np.max(np.abs(np.abs(np.sum(u * uo, axis=0)) - 1)) < 1e-9


def test_evd_symmetric_known_answers_and_rejects(eng):
    e = eng.evd_symmetric(_t(np.diag([5.0, -2.0])))
    assert np.allclose(_np(e.lam), [5, -2], atol=1e-12, rtol=0)
    e = eng.evd_symmetric(_t(np.array([[0.0, 1.0], [1.0, 0.0]])))
    assert np.allclose(_np(e.lam), [1, -1], atol=1e-12, rtol=0)
    assert np.allclose(np.abs(_np(e.U)), 1 / np.sqrt(2), atol=1e-12, rtol=0)
    with pytest.raises(eng.NumericError):
        eng.evd_symmetric(_t(np.array([[1.0, 0.5], [-0.5, 1.0]])))


@pytest.mark.parametrize("m,n,r", [(3, 3, 2), (2, 1, 1), (10, 4, 3), (6, 3, 2), (220, 220, 220),
                                   (4, 9, 2)])
def test_solve_ls_matches_oracle(eng, orc, m, n, r):
    rs = np.random.default_rng(m + 10 * n)
    g = rs.standard_normal((m, n))
    if (m, n) == (6, 3):
        g[:, 2] = g[:, 0]  # rank deficient
    h = rs.standard_normal((m, r))
    x = _np(eng.solve_ls(_t(g), _t(h)))
    xo = orc.solve_ls(g, h)
    assert np.max(np.abs(x - xo)) < 1e-9 * max(1.0, np.max(np.abs(xo)))


@pytest.mark.parametrize("l", [6, 12, 40])
def test_joint_core_matches_stacked_solve(eng, orc, l):
    rs = np.random.default_rng(l)
    g1, h1, g2, h2 = (rs.standard_normal((l, l)) for _ in range(4))
    c = _np(eng.solve_joint_core(_t(g1), _t(h1), _t(g2), _t(h2)))
    c_stacked = orc.solve_joint_core(g1, h1, g2, h2, route=0)
    assert np.max(np.abs(c - c_stacked)) < 1e-9 * max(1.0, np.max(np.abs(c_stacked)))


# -------------------------------------------------------------- pipelines
def _check_svd(f, uo, so, vo, k):
    s = _np(f.sigma)
    assert np.max(np.abs(s[:k] - so[:k]) / so[:k]) < SIG_TOL
    assert max_angle(_np(f.U)[:, :k], uo[:, :k]) < ANG_TOL
    assert max_angle(_np(f.V)[:, :k], vo[:, :k]) < ANG_TOL


@pytest.mark.parametrize("mode,q", [(0, 0), (1, 1), (1, 2), (2, 1), (2, 2)])
def test_rsvd_modes_match_oracle(eng, orc, mode, q):
    sigma = 10.0 ** (-np.arange(400) / 100.0)
    a = haar_test_matrix(800, 400, sigma, 11)
    k, p = 20, 5
    f = eng.rsvd(_t(a), eng.SketchConfig(k, p, q, eng.RangeMode(mode), 1))
    uo, so, vo = orc.rsvd(a, k, p, q, mode, orc.Rng(1))
    _check_svd(f, uo, so, vo, k)


def test_rsvd_config1_full_size(eng, orc):
    """BASELINE configs[0]: Alg 2, 2048 x 1024, sigma_j = 10^-(j-1)/100, k=20 p=5."""
    sigma = 10.0 ** (-np.arange(1024) / 100.0)
    a = haar_test_matrix(2048, 1024, sigma, 1001)
    f = eng.rsvd(_t(a), eng.SketchConfig(20, 5, 0, eng.RangeMode.basic, 1))
    uo, so, vo = orc.rsvd(a, 20, 5, 0, 0, orc.Rng(1))
    _check_svd(f, uo, so, vo, 20)


def test_rsvd_basic_equals_power_q0_bitwise(eng):
    rs = np.random.default_rng(3)
    a = _t(rs.standard_normal((25, 18)))
    f1 = eng.rsvd(a, eng.SketchConfig(5, 3, 7, eng.RangeMode.basic, 11))
    f2 = eng.rsvd(a, eng.SketchConfig(5, 3, 0, eng.RangeMode.power, 11))
    assert np.array_equal(_np(f1.U), _np(f2.U))
    assert np.array_equal(_np(f1.sigma), _np(f2.sigma))
    assert np.array_equal(_np(f1.V), _np(f2.V))


def test_spevd_matches_oracle(eng, orc):
    n = 600
    rs = np.random.default_rng(4)
    u, _ = np.linalg.qr(rs.standard_normal((n, n)))
    lam = np.array([(-1.0) ** j * j ** -1.5 for j in range(1, n + 1)])
    a = (u * lam) @ u.T
    a = np.asfortranarray(0.5 * (a + a.T))
    k, p = 40, 10
    e = eng.spevd_hermitian(_t(a), k, p, eng.Rng(1))
    uo, lo = orc.spevd_hermitian(a, k, p, orc.Rng(1))
    lg = _np(e.lam)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) < SIG_TOL
    assert max_angle(_np(e.U), uo) < ANG_TOL


def test_spevd_counts_one_apply(eng):
    rs = np.random.default_rng(8)
    g = rs.standard_normal((40, 40))
    op = eng.CountingOperator(_t(0.5 * (g + g.T)))
    eng.spevd_hermitian(op, 5, 3, eng.Rng(2))
    assert op.apply_count() == 1 and op.adjoint_count() == 0


def test_spsvd_matches_oracle(eng, orc):
    sigma = np.exp(-np.arange(300) / 40.0)
    a = haar_test_matrix(900, 500, sigma, 21)
    k, p = 30, 10
    f = eng.spsvd_general(_t(a), k, p, eng.Rng(5))
    uo, so, vo = orc.spsvd_general(a, k, p, orc.Rng(5))
    _check_svd(f, uo, so, vo, k)


def test_spsvd_counts_one_apply_one_adjoint(eng):
    rs = np.random.default_rng(9)
    op = eng.CountingOperator(_t(rs.standard_normal((30, 20))))
    eng.spsvd_general(op, 4, 3, eng.Rng(3))
    assert op.apply_count() == 1 and op.adjoint_count() == 1


# ------------------------------------------------------- CUDA-graph replay
def test_graph_replay_matches_eager(eng):
    """Repeated device calls with identical shapes and pointers are captured
    (second call) and replayed as one CUDA graph (third call on).  Every call
    must give bitwise the same factors, RNG state and counter deltas as a
    fresh handle's eager first call, including after a seed change."""
    import ctypes
    import torch
    L = eng._load()
    m, n, k, p, q = 1500, 700, 10, 4, 1
    l = k + p
    a = _t(haar_test_matrix(m, n, np.logspace(0, -3, 40), 5))
    u = torch.empty((l, m), dtype=torch.float64, device="cuda").t()
    v = torch.empty((l, n), dtype=torch.float64, device="cuda").t()
    s = torch.empty(l, dtype=torch.float64, device="cuda")

    def call(e, seed):
        r = eng.Rng(seed)
        c0 = e.counters()
        eng._check(L.rsvd_rsvd_dev(e.handle, m, n, a.data_ptr(), m, k, p, q, 2, ctypes.byref(r.state),
                                   u.data_ptr(), m, s.data_ptr(), v.data_ptr(), n))
        c1 = e.counters()
        d = {key: c1[key] - c0[key] for key in c1}
        return u.cpu().numpy().copy(), s.cpu().numpy().copy(), v.cpu().numpy().copy(), bytes(r.state), d

    e1 = eng.Engine(0)
    runs = [call(e1, 3) for _ in range(4)] + [call(e1, 4)]
    ref3, ref4 = call(eng.Engine(0), 3), call(eng.Engine(0), 4)
    for got, ref in zip(runs, [ref3] * 4 + [ref4]):
        for x, y in zip(got[:3], ref[:3]):
            assert np.array_equal(x, y)
        assert got[3] == ref[3]
        assert got[4] == ref[4]


def test_graph_replay_with_fresh_output_buffers(eng):
    """Graph-cached calls write through workspace staging, so the cache key
    ignores where the caller puts the outputs: calls alternating between
    output buffers (and a padded leading dimension) must each fill their own
    buffers with bitwise the same factors, and leave the other buffers alone."""
    import ctypes
    import torch
    L = eng._load()
    m, n, k, p, q = 1200, 500, 12, 4, 1
    l = k + p
    a = _t(haar_test_matrix(m, n, np.logspace(0, -4, 60), 9))
    e = eng.Engine(0)
    bufs = []
    for ldu in (m, m + 6, m):
        u = torch.full((l, ldu), -7.0, dtype=torch.float64, device="cuda")
        v = torch.full((l, n), -7.0, dtype=torch.float64, device="cuda")
        s = torch.full((l,), -7.0, dtype=torch.float64, device="cuda")
        bufs.append((u, ldu, s, v))

    def call(b):
        u, ldu, s, v = b
        r = eng.Rng(5)
        eng._check(L.rsvd_rsvd_dev(e.handle, m, n, a.data_ptr(), m, k, p, q, 2, ctypes.byref(r.state),
                                   u.data_ptr(), ldu, s.data_ptr(), v.data_ptr(), n))
        torch.cuda.synchronize()
        return u.t()[:m].cpu().numpy().copy(), s.cpu().numpy().copy(), v.t().cpu().numpy().copy()

    ref = call(bufs[0])
    for i in (1, 2, 0, 1, 2, 0):  # eager, capture and replays with changing outputs
        before = [t.clone() for j, b in enumerate(bufs) if j != i for t in (b[0], b[2], b[3])]
        got = call(bufs[i])
        for x, y in zip(got, ref):
            assert np.array_equal(x, y)
        after = [t for j, b in enumerate(bufs) if j != i for t in (b[0], b[2], b[3])]
        for x, y in zip(before, after):
            assert torch.equal(x, y)
    # the padding rows of the padded buffer are untouched
    assert bool((bufs[1][0].t()[m:] == -7.0).all())
