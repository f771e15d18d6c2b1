"""The l x l cores at and beyond the BASELINE sizes (l = 220, 550 and 1500,
reference core.hpp:111-162): svd_small and evd_symmetric on the block-Jacobi
path, whose visits are split over clusters of 1-8 CTAs (bjacobi.cu), against
the oracle (LAPACK dgesdd / dsyevd with the reference's sign and |lambda|
order rules)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a)).cuda().t().contiguous().t()


def _np(t):
    return np.asfortranarray(t.cpu().numpy())


def _svd_check(eng, orc, a, tol_s=1e-12, tol_f=1e-9):
    f = eng.svd_small(_t(a))
    u, s, v = _np(f.U), _np(f.sigma), _np(f.V)
    uo, so, vo = orc.svd_small(a)
    assert np.max(np.abs(s - so) / so) < tol_s
    r = min(a.shape)
    assert np.max(np.abs(u.T @ u - np.eye(r))) < 1e-10
    assert np.max(np.abs(v.T @ v - np.eye(r))) < 1e-10
    # distinct singular values: the sign rule makes the factors comparable
    assert np.max(np.abs(u - uo)) < tol_f
    assert np.max(np.abs(v - vo)) < tol_f


@pytest.mark.parametrize("n,cluster", [(550, 0), (550, 1), (550, 2), (550, 8), (220, 4), (1500, 0),
                                       (837, 0), (97, 0)])
def test_svd_small_large_l(eng, orc, n, cluster):
    """l = 550 (C5's cores) for every cluster size, and l = 837 / 1500, which
    round 1's one-CTA visits could not hold in shared memory."""
    rs = np.random.default_rng(n + cluster)
    u, _ = np.linalg.qr(rs.standard_normal((n, n)))
    v, _ = np.linalg.qr(rs.standard_normal((n, n)))
    a = (u * np.exp(-np.arange(n) / (0.4 * n))) @ v.T
    old = os.environ.get("RSVD_BJ_CLUSTER")
    os.environ["RSVD_BJ_CLUSTER"] = str(cluster)
    try:
        _svd_check(eng, orc, a, tol_s=1e-12, tol_f=1e-8)
    finally:
        if old is None:
            del os.environ["RSVD_BJ_CLUSTER"]
        else:
            os.environ["RSVD_BJ_CLUSTER"] = old


def test_svd_small_wide_1500x2000(eng, orc):
    rs = np.random.default_rng(3)
    a = rs.standard_normal((1500, 2000))
    f = eng.svd_small(_t(a))
    so = orc.svd_small(a)[1]
    assert np.max(np.abs(_np(f.sigma) - so) / so) < 1e-11


@pytest.mark.parametrize("n", [550, 1500])
def test_evd_symmetric_large_l(eng, orc, n):
    rs = np.random.default_rng(n)
    g = rs.standard_normal((n, n))
    c = 0.5 * (g + g.T)
    e = eng.evd_symmetric(_t(c))
    u, lam = _np(e.U), _np(e.lam)
    uo, lo = orc.evd_symmetric(c)
    assert np.max(np.abs(lam - lo)) < 1e-12 * np.max(np.abs(lo))
    assert np.all(np.abs(lam[:-1]) >= np.abs(lam[1:]))
    assert np.max(np.abs(u.T @ u - np.eye(n))) < 1e-10
    # eigenvectors of well-separated eigenvalues agree up to sign
    gap = np.minimum(np.abs(np.diff(lo))[:-1], np.abs(np.diff(lo))[1:])
    sel = np.where(gap > 1e-3 * np.max(np.abs(lo)))[0] + 1
    assert np.max(np.abs(np.abs(np.sum(u[:, sel] * uo[:, sel], axis=0)) - 1)) < 1e-8


def test_svd_small_graded_clustered(eng, orc):
    """A strongly graded 600 x 600 factor takes the one-sided inner route,
    whose dot products are summed over the cluster."""
    rs = np.random.default_rng(11)
    n = 600
    u, _ = np.linalg.qr(rs.standard_normal((n, n)))
    v, _ = np.linalg.qr(rs.standard_normal((n, n)))
    s = 10.0 ** (-np.arange(n) / 40.0)
    a = (u * s) @ v.T
    f = eng.svd_small(_t(a))
    sg = _np(f.sigma)
    so = orc.svd_small(a)[1]
    # A itself carries rounding ~u |A|: both sides are accurate to that
    # absolute level, not relatively, for the values below it
    assert np.max(np.abs(sg - so)) < 1e-12 * so[0]
    ug = _np(f.U)
    assert np.max(np.abs(ug.T @ ug - np.eye(n))) < 1e-10
