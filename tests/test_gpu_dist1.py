"""The row-sharded (multi-GPU) code path on one B200: a handle built over a
one-rank NCCL communicator (rsvd_create_dist with nranks = 1) takes every
branch the sharded engine takes -- distributed CholeskyQR / TSQR with Gram and
R allreduces, n x l and l x l partial allreduces, shard-row allgather -- with
real NCCL calls on the handle's stream.  Its factors must satisfy the same
oracle tolerances as the single-GPU path (the exchange pattern itself is
checked at world size 2 on CPU in test_dist_gloo.py)."""
import numpy as np
import pytest

from test_gpu_parity import ANG_TOL, SIG_TOL, _check_svd, _np, _t, haar_test_matrix, max_angle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dist1(eng):
    e = eng.Engine(0, 0, 1, eng.Engine.nccl_unique_id())
    yield e
    e.close()


def test_one_rank_handle_is_distributed(eng, dist1):
    import ctypes
    r, n = ctypes.c_int(-1), ctypes.c_int(-1)
    assert eng._load().rsvd_dist_info(dist1.handle, ctypes.byref(r), ctypes.byref(n)) == 0
    assert (r.value, n.value) == (0, 1)
    # single-GPU-only diagnostics refuse a distributed handle
    with eng.using_engine(dist1):
        with pytest.raises(eng.ParameterError):
            eng.singular_values(_t(np.eye(8)))


@pytest.mark.parametrize("mode,q,l", [(0, 0, 25), (1, 2, 25), (2, 2, 25), (2, 1, 110)])
def test_rsvd_sharded_path_matches_oracle(eng, orc, dist1, mode, q, l):
    sigma = np.exp(-np.arange(600) / 50.0)
    a = haar_test_matrix(3000, 600, sigma, 31)
    k, p = l - 5 if l <= 32 else l - 10, 5 if l <= 32 else 10
    cfg = eng.SketchConfig(k, p, q, eng.RangeMode(mode), 1)
    with eng.using_engine(dist1):
        dist1.reset_counters()
        f = eng.rsvd(_t(a), cfg)
        c = dist1.counters()
    uo, so, vo = orc.rsvd(a, k, p, q, mode, orc.Rng(1))
    _check_svd(f, uo, so, vo, k)
    assert c["physical_passes"] == 2 * q + 2


def test_spevd_sharded_path_matches_oracle(eng, orc, dist1):
    n = 600
    rs = np.random.default_rng(4)
    u, _ = np.linalg.qr(rs.standard_normal((n, n)))
    lam = np.array([(-1.0) ** j * j ** -1.5 for j in range(1, n + 1)])
    a = (u * lam) @ u.T
    a = np.asfortranarray(0.5 * (a + a.T))
    k, p = 40, 10
    with eng.using_engine(dist1):
        e = eng.spevd_hermitian(_t(a), k, p, eng.Rng(1))
    uo, lo = orc.spevd_hermitian(a, k, p, orc.Rng(1))
    assert np.max(np.abs(_np(e.lam) - lo) / np.abs(lo)) < SIG_TOL
    assert max_angle(_np(e.U), uo) < ANG_TOL


def test_spsvd_sharded_path_matches_oracle(eng, orc, dist1):
    sigma = np.exp(-np.arange(300) / 40.0)
    a = haar_test_matrix(900, 500, sigma, 21)
    k, p = 30, 10
    with eng.using_engine(dist1):
        f = eng.spsvd_general(_t(a), k, p, eng.Rng(5))
    uo, so, vo = orc.spsvd_general(a, k, p, orc.Rng(5))
    _check_svd(f, uo, so, vo, k)


def test_sharded_path_is_deterministic(eng, dist1):
    a = _t(haar_test_matrix(2000, 400, np.logspace(0, -4, 400), 8))
    cfg = eng.SketchConfig(20, 5, 2, eng.RangeMode.power_ortho, 3)
    with eng.using_engine(dist1):
        f1 = eng.rsvd(a, cfg)
        f2 = eng.rsvd(a, cfg)
    assert np.array_equal(_np(f1.sigma), _np(f2.sigma))
    assert np.array_equal(_np(f1.U), _np(f2.U))


def test_sharded_calls_are_graph_captured_and_replayed(eng, dist1):
    """With a shard descriptor the sharded call has no host round trip, so
    repeated calls are captured into a CUDA graph (NCCL collectives
    included) and replayed: every call gives bitwise the first (eager) call's
    factors and the same counter deltas."""
    a = _t(haar_test_matrix(2000, 500, np.exp(-np.arange(500) / 40.0), 33))
    cfg = eng.SketchConfig(20, 5, 2, eng.RangeMode.power, 3)
    dist1.set_shard(2000, 0)
    try:
        outs, deltas = [], []
        with eng.using_engine(dist1):
            for _ in range(4):
                c0 = dist1.counters()
                f = eng.rsvd(a, cfg)
                c1 = dist1.counters()
                outs.append((_np(f.U), _np(f.sigma), _np(f.V)))
                deltas.append({k: c1[k] - c0[k] for k in c1})
        for o, d in zip(outs[1:], deltas[1:]):
            for x, y in zip(o, outs[0]):
                assert np.array_equal(x, y)
            assert d == deltas[0]
    finally:
        dist1.set_shard(0, 0)
