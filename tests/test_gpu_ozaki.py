"""The FP64 pass products on the INT8 tensor cores (csrc/ozaki.cu: tcgen05
kind::i8, Ozaki splitting into S exact 8-bit slices per operand).

Y = A Omega_c and W = A^T Psi of Alg 6 (reference singlepass.hpp:119-122) are
checked against longdouble / fp64 numpy products: with S = 8 slices (62
fractional bits) inside the bound of an fp64 product, |err_ij| <= 2 K u
(|A| |X|)_ij, for every contraction length K; with the default S = 7 (54
fractional bits: the operands are rounded to ~2u of their row / column
maxima before the exact products) inside 2 max(K, 64) u (|A| |X|)_ij -- the
fp64 bound from K = 64 up; with fewer slices inside 2^-(8S-12) of the same
scale.  Edge shapes (ragged tiles, K below one
ring stage, a single row / column), graded and zero rows and columns, row
panels, determinism, and the whole of Alg 6 against the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def _t(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a)).cuda().t().contiguous().t()


@pytest.fixture
def oz(eng):
    yield eng
    eng.set_ozaki_slices(-1)


def _bound(a, x, trans, s):
    k = a.shape[0] if trans else a.shape[1]
    sc = (np.abs(a).T @ np.abs(x)) if trans else (np.abs(a) @ np.abs(x))
    rel = 2 * k * U if s == 8 else 2 * max(k, 64) * U if s == 7 else max(2 * k * U, 2.0 ** -(8 * s - 12))
    return rel * sc + 1e-300


@pytest.fixture(params=[1, 0], ids=["pair", "single"])
def kernel(eng, request):
    """Both GEMM kernels: the CTA pair (cta_group::2, default) and the single CTA."""
    eng.debug_ozaki_kernel(request.param)
    yield request.param
    eng.debug_ozaki_kernel(-1)


@pytest.mark.parametrize("m,n,l", [(300, 200, 25), (1000, 777, 110), (257, 4099, 220), (4100, 130, 30),
                                   (128, 32, 16), (1, 1, 1), (5, 3, 2), (129, 31, 113), (700, 1300, 550)])
@pytest.mark.parametrize("trans", [False, True])
def test_gemm_matches_longdouble_product(eng, kernel, m, n, l, trans):
    rs = np.random.default_rng(m + 3 * n + l)
    a = rs.standard_normal((m, n)) * np.exp(rs.uniform(-3, 3, (m, 1)))
    x = rs.standard_normal((m if trans else n, l))
    ref = (a.T.astype(np.longdouble) @ x.astype(np.longdouble)) if trans else (
        a.astype(np.longdouble) @ x.astype(np.longdouble))
    for s in (8, 7, 5):
        c = eng.debug_ozaki_gemm(_t(a), _t(x), trans=trans, slices=s).cpu().numpy()
        err = np.abs(c - ref).astype(np.float64)
        b = _bound(a, x, trans, s)
        assert np.all(err <= b), (s, float(np.max(err / b)))


def test_gemm_graded_and_zero_rows_columns(eng):
    """Row scales spanning 2^-300..2^300, zero rows of A and zero columns of X:
    the power-of-two scaling is exact, so each output row keeps its own
    relative accuracy."""
    rs = np.random.default_rng(3)
    m, n, l = 500, 300, 40
    a = rs.standard_normal((m, n)) * (2.0 ** rs.integers(-300, 300, (m, 1)))
    a[7] = 0.0
    a[:, 11] = 0.0
    x = rs.standard_normal((n, l))
    x[:, 5] = 0.0
    x[13] = 0.0
    c = eng.debug_ozaki_gemm(_t(a), _t(x), slices=8).cpu().numpy()
    ref = a.astype(np.longdouble) @ x.astype(np.longdouble)
    b = _bound(a, x, False, 8)
    assert np.all(np.abs(c - ref).astype(np.float64) <= b)
    assert np.all(c[7] == 0.0) and np.all(c[:, 5] == 0.0)
    # adjoint: the rows' scales move into the skinny operand
    y = rs.standard_normal((m, l))
    a2 = rs.standard_normal((m, n)) * (2.0 ** rs.integers(-30, 30, (m, 1)))
    c2 = eng.debug_ozaki_gemm(_t(a2), _t(y), trans=True, slices=8).cpu().numpy()
    ref2 = a2.T.astype(np.longdouble) @ y.astype(np.longdouble)
    assert np.all(np.abs(c2 - ref2).astype(np.float64) <= _bound(a2, y, True, 8))


def test_gemm_very_wide_matrix(eng):
    """More than 65535 * 8 columns of A: the slicing grid puts columns on grid.x."""
    rs = np.random.default_rng(2)
    m, n, l = 40, 600000, 3
    a = rs.standard_normal((m, n))
    x = rs.standard_normal((n, l))
    c = eng.debug_ozaki_gemm(_t(a), _t(x), slices=8).cpu().numpy()
    assert np.all(np.abs(c - a @ x) <= 2 * _bound(a, x, False, 8))
    y = rs.standard_normal((m, l))
    c2 = eng.debug_ozaki_gemm(_t(a), _t(y), trans=True, slices=8).cpu().numpy()
    assert np.all(np.abs(c2 - a.T @ y) <= 2 * _bound(a, y, True, 8))


def test_gemm_long_contraction_chunks(eng, kernel):
    """Contractions longer than 16384 steps: the kernels drain their int32
    accumulators to fp64 every 16384 steps (8192 with 8 slices)."""
    rs = np.random.default_rng(8)
    m, n, l = 130, 70000, 20
    a = rs.standard_normal((m, n))
    x = rs.standard_normal((n, l))
    ref = a.astype(np.longdouble) @ x.astype(np.longdouble)
    for s in (8, 7):
        c = eng.debug_ozaki_gemm(_t(a), _t(x), slices=s).cpu().numpy()
        assert np.all(np.abs(c - ref).astype(np.float64) <= _bound(a, x, False, s))
    y = rs.standard_normal((n, 7))  # adjoint: contraction over 70000 rows (sub-panels and chunks)
    c = eng.debug_ozaki_gemm(_t(a.T.copy()), _t(y), trans=True, slices=7).cpu().numpy()
    refa = a.astype(np.longdouble) @ y.astype(np.longdouble)
    assert np.all(np.abs(c - refa).astype(np.float64) <= _bound(a.T, y, True, 7))
    # extreme digits: every entry at the top of its slice range
    a1 = np.full((m, 40000), 1.0 - 2.0 ** -52)
    x1 = np.full((40000, 3), -(1.0 - 2.0 ** -52))
    c1 = eng.debug_ozaki_gemm(_t(a1), _t(x1), slices=8).cpu().numpy()
    assert np.allclose(c1, a1 @ x1, rtol=1e-13, atol=0)


@pytest.mark.parametrize("m,n,l,panel", [(3000, 700, 30, 256), (4096, 1024, 70, 1000), (300, 5000, 550, 0),
                                         (2049, 4095, 57, 2048)])
def test_dual_pass_on_int8_tensor_cores(oz, m, n, l, panel):
    rs = np.random.default_rng(m + n + l)
    a, oc, psi = rs.standard_normal((m, n)), rs.standard_normal((n, l)), rs.standard_normal((m, l))
    oz.set_ozaki_slices(8)
    y, w = oz.debug_dual_pass(_t(a), _t(oc), _t(psi), panel_rows=panel)
    y2, w2 = oz.debug_dual_pass(_t(a), _t(oc), _t(psi), panel_rows=panel)
    assert np.array_equal(y.cpu().numpy(), y2.cpu().numpy())  # deterministic
    assert np.array_equal(w.cpu().numpy(), w2.cpu().numpy())
    y, w = y.cpu().numpy(), w.cpu().numpy()
    assert np.all(np.abs(y - a @ oc) <= 2 * _bound(a, oc, False, 8))
    assert np.all(np.abs(w - a.T @ psi) <= 2 * _bound(a, psi, True, 8))


@pytest.mark.parametrize("slices", [8, 7, 6])
def test_spsvd_on_int8_tensor_cores_matches_oracle(oz, orc, slices):
    """Alg 6 end to end with the sliced pass: north-star tolerances vs the
    oracle, one physical pass counted, host-streamed call included."""
    rs = np.random.default_rng(12)
    m, n, r = 6000, 1500, 60
    u, _ = np.linalg.qr(rs.standard_normal((m, r)))
    v, _ = np.linalg.qr(rs.standard_normal((n, r)))
    a = np.asfortranarray((u * np.exp(-np.arange(r) / 10.0)) @ v.T + 1e-9 * rs.standard_normal((m, n)))
    k, p = 30, 10
    oz.set_ozaki_slices(slices)
    op = oz.CountingOperator(_t(a))
    f = oz.spsvd_general(op, k, p, oz.Rng(4))
    assert op.apply_count() == 1 and op.adjoint_count() == 1 and op.physical_passes() == 1
    uo, so, vo = orc.spsvd_general(a, k, p, orc.Rng(4))
    sg = f.sigma.cpu().numpy()
    assert np.max(np.abs(sg[:k] - so[:k]) / so[:k]) < 1e-10
    for g, o in ((f.U.cpu().numpy(), uo), (f.V.cpu().numpy(), vo)):
        s = np.linalg.svd(g[:, :k] - o[:, :k] @ (o[:, :k].T @ g[:, :k]), compute_uv=False)[0]
        assert np.arcsin(min(1.0, s)) < 1e-8
    fh = oz.spsvd_general(a, k, p, oz.Rng(4))  # pinned-host path, row panels
    assert np.max(np.abs(np.asarray(fh.sigma)[:k] - so[:k]) / so[:k]) < 1e-10


@pytest.mark.parametrize("mode,q", [("basic", 0), ("power", 1), ("power_ortho", 2)])
def test_rsvd_passes_on_int8_tensor_cores_match_oracle(oz, orc, mode, q):
    """Algs 2-4 with every product A X / A^T Y on the sliced INT8 path (A's
    slices built once per call and reused by the 2q + 2 passes)."""
    rs = np.random.default_rng(21)
    m, n, k, p = 3000, 2000, 30, 10
    u, _ = np.linalg.qr(rs.standard_normal((m, n)))
    v, _ = np.linalg.qr(rs.standard_normal((n, n)))
    a = np.asfortranarray((u * np.exp(-np.arange(n) / 20.0)) @ v.T)
    oz.set_ozaki_slices(8)
    f = oz.rsvd(_t(a), oz.SketchConfig(k, p, q, oz.RangeMode[mode], 5))
    uo, so, vo = orc.rsvd(a, k, p, q, {"basic": 0, "power": 1, "power_ortho": 2}[mode], orc.Rng(5))
    sg = f.sigma.cpu().numpy()
    assert np.max(np.abs(sg[:k] - so[:k]) / so[:k]) < 1e-10
    for g, o in ((f.U.cpu().numpy(), uo), (f.V.cpu().numpy(), vo)):
        s = np.linalg.svd(g[:, :k] - o[:, :k] @ (o[:, :k].T @ g[:, :k]), compute_uv=False)[0]
        assert np.arcsin(min(1.0, s)) < 1e-8
    c = oz.default_engine().counters()
    assert c["kernel_launches"] > 0


def test_non_finite_inputs_raise_numeric_error_on_int8_path(oz):
    """Inf / NaN cannot be sliced; the exponent scans flag them and the call
    ends in NumericError like the FP64 passes (core.hpp:36-39)."""
    rs = np.random.default_rng(0)
    a = rs.standard_normal((400, 300))
    oz.set_ozaki_slices(8)
    for bad in (np.nan, np.inf, -np.inf):
        b = a.copy()
        b[17, 23] = bad
        with pytest.raises(oz.NumericError):
            oz.rsvd(_t(b), oz.SketchConfig(5, 2, 1, oz.RangeMode.power, 1))
        with pytest.raises(oz.NumericError):
            oz.spsvd_general(_t(b), 5, 2, oz.Rng(1))
    f = oz.spsvd_general(_t(a), 5, 2, oz.Rng(1))  # the engine stays usable
    assert np.isfinite(f.sigma.cpu().numpy()).all()


@pytest.mark.slow
def test_c5_size_pass_int8_agrees_with_dmma(oz):
    """BASELINE C5's full-size dual pass (A 262144 x 32768, l = 550) on both
    arithmetic paths: the INT8 tensor-core products and the FP64 DMMA fused
    pass agree entrywise within the sum of their fp64 error bounds, with
    (|A||X|)_ij bounded by ||a_i||_2 ||x_j||_2 (no second 68.7 GB matrix)."""
    import torch
    import bench
    cfg = bench.CONFIGS["C5"]
    dev = torch.device("cuda", 0)
    a = bench.make_input(cfg, dev)
    m, n = a.shape
    l = cfg["k"] + cfg["p"]
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    oc = torch.randn((l, n), dtype=torch.float64, device=dev, generator=g).t()
    psi = torch.randn((l, m), dtype=torch.float64, device=dev, generator=g).t()
    oz.set_ozaki_slices(7)
    y8, w8 = oz.debug_dual_pass(a, oc, psi)
    oz.set_ozaki_slices(0)
    yd, wd = oz.debug_dual_pass(a, oc, psi)
    rown = torch.linalg.vector_norm(a, dim=1)
    coln = torch.linalg.vector_norm(a, dim=0)
    by = 4 * n * U * rown[:, None] * torch.linalg.vector_norm(oc, dim=0)[None, :]
    bw = 4 * m * U * coln[:, None] * torch.linalg.vector_norm(psi, dim=0)[None, :]
    ry = float(((y8 - yd).abs() / by).max())
    rw = float(((w8 - wd).abs() / bw).max())
    print(f"C5-size pass: max |Y8 - Yd| / bound {ry:.3e}, max |W8 - Wd| / bound {rw:.3e}; "
          f"relative to max|Y| {float((y8 - yd).abs().max() / yd.abs().max()):.3e}")
    assert ry <= 1.0 and rw <= 1.0


def test_set_ozaki_slices_rejects_bad_values(oz):
    with pytest.raises(oz.ParameterError):
        oz.set_ozaki_slices(2)
    with pytest.raises(oz.ParameterError):
        oz.set_ozaki_slices(9)
