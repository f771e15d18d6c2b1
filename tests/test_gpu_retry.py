"""Speculative CholeskyQR (small.cu cholqr): without a host round trip the
engine assumes its sketch needs no shifted Cholesky; when one does (a
numerically rank-deficient sketch) a device flag makes the call re-run in
robust mode -- counted in `robust_reruns` -- and the result is the robust
path's.  Well-conditioned calls never re-run (bitwise the robust result)."""
import numpy as np
import pytest

from test_gpu_parity import _np, _t, haar_test_matrix

pytestmark = pytest.mark.gpu


def test_rank_deficient_orthonormalize_reruns_robustly(eng, orc):
    rs = np.random.default_rng(5)
    x = rs.standard_normal((3000, 60)) @ rs.standard_normal((60, 100))  # rank 60 of 100 columns
    e = eng.default_engine()
    for rep in range(3):  # eager, captured, replayed
        c0 = e.counters()
        q = _np(eng.orthonormalize(_t(x)))
        c1 = e.counters()
        assert c1["robust_reruns"] - c0["robust_reruns"] == 1
        assert np.max(np.abs(q.T @ q - np.eye(100))) < 1e-12
        # the basis spans x: the residual of x projected out is at rounding
        r = x - q @ (q.T @ x)
        assert np.linalg.norm(r) < 1e-11 * np.linalg.norm(x)


def test_well_conditioned_calls_do_not_rerun(eng):
    a = _t(haar_test_matrix(4000, 1000, np.exp(-np.arange(1000) / 100.0), 12))
    e = eng.default_engine()
    cfg = eng.SketchConfig(90, 10, 1, eng.RangeMode.power_ortho, 4)  # l = 100: the l > 64 CholeskyQR
    c0 = e.counters()
    for _ in range(3):
        eng.rsvd(a, cfg)
    c1 = e.counters()
    assert c1["robust_reruns"] == c0["robust_reruns"]
