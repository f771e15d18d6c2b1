"""The row-sharded (multi-GPU) engine with P = 2, 3 and 8 ranks, run on ONE
GPU through the virtual communicator (rsvd_create_virtual, dist.cu): one
thread and one handle per rank, fixed-order device reductions instead of
NCCL.  Everything above the collectives is the code an 8-GPU job runs: shard
offsets, Psi row selection, the distributed CholeskyQR / TSQR, the n x l and
l x l allreduces, the fused Alg-6 pass on each shard, and Alg 5's sharded
asymmetry precondition (blocks exchanged rank to rank).

Each rank factors its np.array_split row block; the assembled factors are
compared with the oracle on the whole matrix at the north-star tolerances
(sigma / |lambda| 1e-10 relative, canonical angles 1e-8 rad), and the
replicated outputs must be bitwise equal on every rank."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIG_TOL, ANG_TOL = 1e-10, 1e-8


def _t(a):
    import torch
    return torch.from_numpy(np.asfortranarray(a)).cuda().t().contiguous().t()


def sin_max(x, y):
    r = y - x @ (x.T @ y)
    return float(np.linalg.svd(r, compute_uv=False)[0])


def haar_matrix(m, n, sigma, seed):
    rs = np.random.default_rng(seed)
    u, r = np.linalg.qr(rs.standard_normal((m, len(sigma))))
    v, r2 = np.linalg.qr(rs.standard_normal((n, len(sigma))))
    return np.asfortranarray((u * sigma) @ v.T)


def _shards(a, nranks):
    return [_t(a[idx, :]) for idx in np.array_split(np.arange(a.shape[0]), nranks)]


@pytest.fixture(scope="module")
def vcomms(eng):
    made = {}

    def get(p):
        if p not in made:
            made[p] = eng.VirtualComm(p)
        return made[p]
    yield get
    for v in made.values():
        v.close()


def _assemble(parts):
    u = np.vstack([p[0] for p in parts])
    for p in parts[1:]:  # replicated outputs: bitwise equal on every rank
        assert np.array_equal(p[1], parts[0][1])
        if p[2] is not None:
            assert np.array_equal(p[2], parts[0][2])
    return u, parts[0][1], parts[0][2]


@pytest.mark.parametrize("nranks", [2, 3, 8])
@pytest.mark.parametrize("mode,q", [(0, 0), (1, 2), (2, 2)])
def test_sharded_rsvd_matches_oracle(eng, orc, vcomms, nranks, mode, q):
    """Alg 2 / 3 / 4 on P row shards."""
    a = haar_matrix(1000, 600, 10.0 ** (-np.arange(600) / 100.0), 7)
    k, p = 20, 5
    shards = _shards(a, nranks)

    def run(r, e):
        f = eng.rsvd(shards[r], eng.SketchConfig(k, p, q, eng.RangeMode(mode), 1))
        return f.U.cpu().numpy(), f.sigma.cpu().numpy(), f.V.cpu().numpy()
    u, s, v = _assemble(vcomms(nranks).run(run))
    uo, so, vo = orc.rsvd(a, k, p, q, mode, orc.Rng(1))
    assert np.max(np.abs(s[:k] - so[:k]) / so[:k]) < SIG_TOL
    assert sin_max(u[:, :k], uo[:, :k]) < ANG_TOL
    assert sin_max(v[:, :k], vo[:, :k]) < ANG_TOL


@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_sharded_spsvd_matches_oracle(eng, orc, vcomms, nranks):
    """Alg 6: each rank's fused pass over its shard, Psi's local rows from the
    replicated stream, W = sum of the shards' A^T Psi partials."""
    a = haar_matrix(1500, 700, np.exp(-np.arange(200) / 30.0), 8)
    k, p = 30, 10
    shards = _shards(a, nranks)

    def run(r, e):
        f = eng.spsvd_general(shards[r], k, p, eng.Rng(5))
        return f.U.cpu().numpy(), f.sigma.cpu().numpy(), f.V.cpu().numpy()
    u, s, v = _assemble(vcomms(nranks).run(run))
    uo, so, vo = orc.spsvd_general(a, k, p, orc.Rng(5))
    assert np.max(np.abs(s[:k] - so[:k]) / so[:k]) < SIG_TOL
    assert sin_max(u[:, :k], uo[:, :k]) < ANG_TOL
    assert sin_max(v[:, :k], vo[:, :k]) < ANG_TOL


@pytest.mark.parametrize("nranks", [2, 3])
def test_sharded_int8_passes_match_oracle(eng, orc, vcomms, nranks):
    """The INT8 tensor-core passes (csrc/ozaki.cu) on row shards: every rank
    slices its own rows (row exponents are local, Psi's local rows carry
    them), the partial W / Z are allreduced as on the DMMA path.  Alg 6 and
    Alg 4 against the oracle, replicated outputs bitwise equal on all ranks."""
    a = haar_matrix(1500, 700, np.exp(-np.arange(200) / 30.0), 8)
    k, p = 30, 10
    shards = _shards(a, nranks)

    def run6(r, e):
        eng.set_ozaki_slices(8, e)
        try:
            f = eng.spsvd_general(shards[r], k, p, eng.Rng(5))
        finally:
            eng.set_ozaki_slices(-1, e)
        return f.U.cpu().numpy(), f.sigma.cpu().numpy(), f.V.cpu().numpy()
    u, s, v = _assemble(vcomms(nranks).run(run6))
    uo, so, vo = orc.spsvd_general(a, k, p, orc.Rng(5))
    assert np.max(np.abs(s[:k] - so[:k]) / so[:k]) < SIG_TOL
    assert sin_max(u[:, :k], uo[:, :k]) < ANG_TOL
    assert sin_max(v[:, :k], vo[:, :k]) < ANG_TOL

    def run4(r, e):
        eng.set_ozaki_slices(8, e)
        try:
            f = eng.rsvd(shards[r], eng.SketchConfig(k, p, 2, eng.RangeMode(2), 1))
        finally:
            eng.set_ozaki_slices(-1, e)
        return f.U.cpu().numpy(), f.sigma.cpu().numpy(), f.V.cpu().numpy()
    u, s, v = _assemble(vcomms(nranks).run(run4))
    uo, so, vo = orc.rsvd(a, k, p, 2, 2, orc.Rng(1))
    assert np.max(np.abs(s[:k] - so[:k]) / so[:k]) < SIG_TOL
    assert sin_max(u[:, :k], uo[:, :k]) < ANG_TOL
    assert sin_max(v[:, :k], vo[:, :k]) < ANG_TOL


def _sym(n, seed):
    rs = np.random.default_rng(seed)
    uq, _ = np.linalg.qr(rs.standard_normal((n, n)))
    lam = np.array([(-1.0) ** j * j ** -1.5 for j in range(1, n + 1)])
    a = (uq * lam) @ uq.T
    return np.asfortranarray(0.5 * (a + a.T))


@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_sharded_spevd_matches_oracle(eng, orc, vcomms, nranks):
    """Alg 5 on row shards of a square A (m_global == n), with the sharded
    asymmetry precondition."""
    a = _sym(640, 4)
    k, p = 30, 10
    shards = _shards(a, nranks)

    def run(r, e):
        f = eng.spevd_hermitian(shards[r], k, p, eng.Rng(1))
        return f.U.cpu().numpy(), f.lam.cpu().numpy(), None
    u, lam, _ = _assemble(vcomms(nranks).run(run))
    uo, lo = orc.spevd_hermitian(a, k, p, orc.Rng(1))
    assert np.max(np.abs(lam - lo) / np.abs(lo)) < SIG_TOL
    assert sin_max(u, uo) < ANG_TOL


@pytest.mark.parametrize("nranks", [2, 3])
def test_sharded_spevd_rejects_asymmetric(eng, vcomms, nranks):
    """One off-diagonal entry on one rank breaks symmetry: every rank raises
    the reference's NumericError (singlepass.hpp:49-53)."""
    a = _sym(300, 6)
    a[250, 3] += 1e-3  # row 250 lives on the last rank, its mirror on rank 0
    shards = _shards(a, nranks)
    errs = []

    def run(r, e):
        try:
            eng.spevd_hermitian(shards[r], 5, 3, eng.Rng(1))
        except eng.NumericError as ex:
            errs.append(str(ex))
        return None
    vcomms(nranks).run(run)
    assert len(errs) == nranks and all("symmetric" in m for m in errs)


def test_sharded_runs_are_deterministic(eng, vcomms):
    a = haar_matrix(900, 400, 10.0 ** (-np.arange(400) / 80.0), 9)
    shards = _shards(a, 3)

    def run(r, e):
        f = eng.rsvd(shards[r], eng.SketchConfig(10, 5, 1, eng.RangeMode.power_ortho, 2))
        return f.U.cpu().numpy(), f.sigma.cpu().numpy(), f.V.cpu().numpy()
    x = _assemble(vcomms(3).run(run))
    y = _assemble(vcomms(3).run(run))
    for p, q in zip(x, y):
        assert np.array_equal(p, q)


def test_sharded_counts_match_single_gpu(eng, vcomms):
    """Every rank counts the same applications and physical passes as the
    single-GPU engine (the exchanges are not passes over A)."""
    a = haar_matrix(800, 300, np.exp(-np.arange(100) / 10.0), 10)
    shards = _shards(a, 2)

    def run(r, e):
        e.reset_counters()
        eng.spsvd_general(shards[r], 8, 4, eng.Rng(3))
        c1 = e.counters()
        e.reset_counters()
        eng.rsvd(shards[r], eng.SketchConfig(8, 4, 2, eng.RangeMode.power, 3))
        c2 = e.counters()
        return c1, c2
    for c1, c2 in vcomms(2).run(run):
        assert (c1["apply"], c1["adjoint"], c1["physical_passes"]) == (1, 1, 1)
        assert (c2["apply"], c2["adjoint"], c2["physical_passes"]) == (3, 3, 6)


@pytest.mark.parametrize("nranks", [2, 3])
def test_sharded_host_entry_points(eng, orc, vcomms, nranks):
    """The host-buffer single-pass calls on row shards (what bench.py's e2e
    leg runs under torchrun): each rank streams its shard up in row panels."""
    a = _sym(600, 12)
    k, p = 20, 8
    idx = np.array_split(np.arange(a.shape[0]), nranks)

    def run(r, e):
        f = eng.spevd_host(np.asfortranarray(a[idx[r], :]), k, p, eng.Rng(1))
        return np.asarray(f.U), np.asarray(f.lam), None
    u, lam, _ = _assemble(vcomms(nranks).run(run))
    uo, lo = orc.spevd_hermitian(a, k, p, orc.Rng(1))
    assert np.max(np.abs(lam - lo) / np.abs(lo)) < SIG_TOL
    assert sin_max(u, uo) < ANG_TOL
    b = haar_matrix(1200, 500, np.exp(-np.arange(150) / 25.0), 13)
    idx = np.array_split(np.arange(b.shape[0]), nranks)

    def run2(r, e):
        f = eng.spsvd_host(np.asfortranarray(b[idx[r], :]), k, p, eng.Rng(2))
        return np.asarray(f.U), np.asarray(f.sigma), np.asarray(f.V)
    u, s, v = _assemble(vcomms(nranks).run(run2))
    uo, so, vo = orc.spsvd_general(b, k, p, orc.Rng(2))
    assert np.max(np.abs(s[:k] - so[:k]) / so[:k]) < SIG_TOL
    assert sin_max(u[:, :k], uo[:, :k]) < ANG_TOL
    assert sin_max(v[:, :k], vo[:, :k]) < ANG_TOL
