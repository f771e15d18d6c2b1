"""Alg 6's fused single pass (fused.cu): Y = A Omega_c and W = A^T Psi from
one traversal of A (reference singlepass.hpp:119-122).

Checked against fp64 numpy products with the summation error bound
|err_ij| <= 2 K u (|A| |X|)_ij (K = the contraction length), for edge shapes
(partial macroblocks, l not a multiple of the 56-column tile, K < one
macroblock), several macroblock edges and row-panel launch sequences (the
streamed host path).  The in-place ordered accumulation is deterministic:
repeated runs, and panelled vs single launches, are bitwise equal."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def _t(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a)).cuda().t().contiguous().t()


def _check(a, oc, psi, y, w):
    y = y.cpu().numpy()
    w = w.cpu().numpy()
    m, n = a.shape
    yr = a @ oc
    wr = a.T @ psi
    by = 2 * n * U * (np.abs(a) @ np.abs(oc)) + 1e-300
    bw = 2 * m * U * (np.abs(a).T @ np.abs(psi)) + 1e-300
    assert np.all(np.abs(y - yr) <= by), np.max(np.abs(y - yr) / by)
    assert np.all(np.abs(w - wr) <= bw), np.max(np.abs(w - wr) / bw)


@pytest.mark.parametrize("m,n,l,mb", [
    (1000, 700, 6, 0), (4096, 2048, 64, 0), (3000, 5000, 110, 0), (2049, 4095, 57, 0),
    (64, 64, 1, 0), (130, 3, 5, 0), (700, 1300, 25, 64), (1500, 900, 113, 128),
    (5000, 300, 56, 256), (300, 5000, 550, 0)])
def test_dual_pass_matches_products(eng, m, n, l, mb):
    rs = np.random.default_rng(m * 7 + n + l)
    a = rs.standard_normal((m, n))
    oc = rs.standard_normal((n, l))
    psi = rs.standard_normal((m, l))
    y, w = eng.debug_dual_pass(_t(a), _t(oc), _t(psi), macroblock=mb)
    _check(a, oc, psi, y, w)


@pytest.mark.parametrize("m,n,l,mb,panel", [(3000, 700, 30, 128, 256), (4096, 1024, 70, 256, 1000),
                                            (2048, 2048, 25, 0, 2048)])
def test_dual_pass_panels_bitwise_equal_single_launch(eng, m, n, l, mb, panel):
    """The streamed host path issues one launch per row panel; the W tiles
    still accumulate macroblock rows in increasing order, so the result is
    bitwise the single launch's, and repeated runs are bitwise equal."""
    rs = np.random.default_rng(5)
    a, oc, psi = _t(rs.standard_normal((m, n))), _t(rs.standard_normal((n, l))), _t(rs.standard_normal((m, l)))
    y1, w1 = eng.debug_dual_pass(a, oc, psi, macroblock=mb)
    y2, w2 = eng.debug_dual_pass(a, oc, psi, macroblock=mb)
    y3, w3 = eng.debug_dual_pass(a, oc, psi, panel_rows=panel, macroblock=mb)
    for x, z in [(y1, y2), (w1, w2), (y1, y3), (w1, w3)]:
        assert np.array_equal(x.cpu().numpy(), z.cpu().numpy())
    _check(a.cpu().numpy(), oc.cpu().numpy(), psi.cpu().numpy(), y1, w1)


def test_spsvd_one_physical_pass(eng):
    """Alg 6 reads A once: one apply, one adjoint, ONE physical pass."""
    rs = np.random.default_rng(9)
    op = eng.CountingOperator(_t(rs.standard_normal((300, 200))))
    eng.spsvd_general(op, 4, 3, eng.Rng(3))
    assert op.apply_count() == 1 and op.adjoint_count() == 1
    assert op.physical_passes() == 1


def test_spsvd_host_streamed_equals_device(eng):
    """The host entry point streams A in row panels into the fused pass as
    they land; the factors are bitwise those of the device-pointer call."""
    rs = np.random.default_rng(12)
    m, n = 9000, 1500
    u, _ = np.linalg.qr(rs.standard_normal((m, 60)))
    v, _ = np.linalg.qr(rs.standard_normal((n, 60)))
    a = np.asfortranarray((u * np.exp(-np.arange(60) / 10.0)) @ v.T + 1e-9 * rs.standard_normal((m, n)))
    fd = eng.spsvd_general(_t(a), 30, 10, eng.Rng(4))
    fh = eng.spsvd_general(a, 30, 10, eng.Rng(4))
    assert np.array_equal(fd.sigma.cpu().numpy(), np.asarray(fh.sigma))
    assert np.array_equal(fd.U.cpu().numpy(), np.asarray(fh.U))
    assert np.array_equal(fd.V.cpu().numpy(), np.asarray(fh.V))


def test_spevd_host_streamed_matches_oracle(eng, orc):
    """Alg 5's host entry point streams A in row panels (apply per panel as
    it lands; the asymmetry precondition once all panels are resident)."""
    rs = np.random.default_rng(4)
    n = 5000
    q, _ = np.linalg.qr(rs.standard_normal((n, 80)))
    lam = np.array([(-1.0) ** j * j ** -1.5 for j in range(1, 81)])
    a = (q * lam) @ q.T
    a = np.asfortranarray(0.5 * (a + a.T))
    e = eng.spevd_hermitian(a, 40, 10, eng.Rng(1))
    uo, lo = orc.spevd_hermitian(a, 40, 10, orc.Rng(1))
    lg = np.asarray(e.lam)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) < 1e-10
    ug = np.asarray(e.U)
    s = np.linalg.svd(ug - uo @ (uo.T @ ug), compute_uv=False)[0]
    assert np.arcsin(min(1.0, s)) < 1e-8


def test_spevd_host_rejects_asymmetric(eng):
    rs = np.random.default_rng(2)
    a = np.asfortranarray(rs.standard_normal((3000, 3000)))
    with pytest.raises(eng.NumericError):
        eng.spevd_hermitian(a, 5, 3, eng.Rng(1))
