"""Multi-GPU sharding logic, exercised on CPU with world_size 2 over gloo.

The engine row-shards A (dist.cu / engine.cu): products with A are local, and
only these exchanges cross ranks:
  * A^T Y partials (n x l)                        -> allreduce   (op_adjoint)
  * CholeskyQR Gram partials (l x l)              -> allreduce   (small.cu cholqr, dist)
  * per-rank TSQR R factors (l x l)               -> allgather   (small.cu tsqr, dist)
  * Alg 5/6 inner products Q^T Omega, Psi^T Q_c   -> allreduce
  * shard sizes                                   -> allgather   (shard_rows)
This test replays exactly that decomposition with numpy + torch.distributed
(gloo) and checks it reproduces the single-process oracle's factorization,
and that bench.py's row partition matches the engine's row offsets.  CPU only.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def _allgather(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.numpy() for o in out]


def _householder_q(x):
    q, r = np.linalg.qr(x)
    return q, r


def dist_tsqr(y_loc):
    """small.cu tsqr(dist=True): local QR, allgather R, QR of the stack, seed
    the local Q with this rank's rows of the stacked Q."""
    q_loc, r_loc = _householder_q(y_loc)
    rs = _allgather(r_loc)
    l = y_loc.shape[1]
    q_s, r_top = _householder_q(np.vstack(rs))
    c = q_s[dist.get_rank() * l:(dist.get_rank() + 1) * l]
    return q_loc @ c, r_top


def dist_cholqr(y_loc, m_global, passes=4):
    """small.cu cholqr(dist=True): per pass the l x l Gram partials are
    allreduced, then the (replicated) Cholesky, shifted by
    11 (m l + l (l+1)) u tr(G) when a pivot loses all precision, and
    Q_loc = Y_loc R^-1.  4 passes for l <= 64 (shifted CholeskyQR3 + 1)."""
    q = y_loc
    l = y_loc.shape[1]
    coef = 11.0 * (m_global * l + l * (l + 1)) * 1.1102230246251565e-16
    for _ in range(passes):
        g = _allreduce(q.T @ q)
        try:
            L = np.linalg.cholesky(g)
            if np.any(np.diag(L) ** 2 <= 1e-12 * np.diag(g)):
                raise np.linalg.LinAlgError
        except np.linalg.LinAlgError:
            L = np.linalg.cholesky(g + coef * np.trace(g) * np.eye(l))
        q = q @ np.linalg.inv(L.T)
    return q


def _worker(rank, world, port, a, omega, res_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = a.shape[0]
    # bench.py partition; shard_rows offsets = prefix sums of m_local
    rows = np.array_split(np.arange(m), world)[rank]
    r0, r1 = int(rows[0]), int(rows[-1]) + 1
    sizes = _allgather(np.array([r1 - r0], dtype=np.float64))
    assert r0 == int(sum(s[0] for s in sizes[:rank]))
    a_loc = a[r0:r1]
    # Alg 3 (rangefinder.hpp:70-79) sharded: Y_g = A_g Omega; Z = sum A_g^T Y_g
    y = a_loc @ omega
    for _ in range(2):
        z = _allreduce(a_loc.T @ y)
        y = a_loc @ z
    q_loc = dist_cholqr(y, m)  # kappa(Y) ~ 1e6 here: the shifted passes engage
    # Stage 2 (factor.hpp:14-16): B^T = sum A_g^T Q_g, replicated small SVD
    z = _allreduce(a_loc.T @ q_loc)
    u_b, s, vt = np.linalg.svd(z.T, full_matrices=False)
    u_loc = q_loc @ u_b
    mx = -(-m // world)  # all_gather needs equal sizes: pad the row shards
    pad = np.zeros((mx, u_loc.shape[1]))
    pad[:r1 - r0] = u_loc
    u_all = [g[:int(s[0])] for g, s in zip(_allgather(pad), sizes)]
    q2 = dist_cholqr(a_loc @ omega, m)
    gram = _allreduce(q2.T @ q2)
    q3, _ = dist_tsqr(a_loc @ omega)  # the row-sharded TSQR variant (R allgather)
    gram3 = _allreduce(q3.T @ q3)
    assert np.max(np.abs(gram3 - np.eye(gram3.shape[0]))) < 1e-12
    if rank == 0:
        np.savez(res_path, s=s, v=vt.T, u=np.vstack(u_all), gram=gram)
    dist.destroy_process_group()


def test_row_sharded_alg3_matches_single_process(orc, tmp_path):
    rs = np.random.default_rng(0)
    m, n, k, p = 301, 120, 8, 4
    u, _ = np.linalg.qr(rs.standard_normal((m, n)))
    v, _ = np.linalg.qr(rs.standard_normal((n, n)))
    sig = 2.0 ** (-np.arange(n) / 4.0)
    a = (u * sig) @ v.T
    omega = orc.gaussian(n, k + p, orc.Rng(1))
    res = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), a, omega, res), nprocs=2, join=True)
    got = np.load(res)
    uo, so, vo = orc.rsvd(np.asfortranarray(a), k, p, 2, orc.POWER, orc.Rng(1))
    assert np.max(np.abs(got["s"][:k] - so[:k]) / so[:k]) < 1e-10
    for x, y in ((got["u"][:, :k], uo[:, :k]), (got["v"][:, :k], vo[:, :k])):
        sin = np.linalg.svd(y - x @ (x.T @ y), compute_uv=False)[0]
        assert sin < 1e-8
    assert np.max(np.abs(got["gram"] - np.eye(k + p))) < 1e-12
