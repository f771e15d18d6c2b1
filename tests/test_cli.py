"""`rsvd-b200 svd` (paper_2402_17794_b200/cli/rsvd_b200_svd.cpp): the
reference's `rsvd svd` command (drivers.hpp:110-175) on the GPU path
(SURVEY §8(f) row 2).  Usage / I/O errors and their exit codes (drivers.hpp:
56-61) are checked on CPU; the factorization and the error report against
the oracle need the GPU."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2402_17794_b200", "lib", "rsvd-b200")


def run(*args):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300)


def test_cli_built():
    assert os.access(CLI, os.X_OK)


@pytest.mark.parametrize("args,code", [((), 2), (("svd",), 2), (("svd", "--k", "3"), 2),
                                       (("svd", "--in", "x.npy"), 2),
                                       (("svd", "--in", "x.npy", "--k", "3", "--alg", "nope"), 2),
                                       (("svd", "--in", "/nonexistent/a.npy", "--k", "3"), 3),
                                       (("svd", "--in", "x.npy", "--k", "two"), 2)])
def test_cli_usage_and_io_errors(args, code):
    r = run(*args)
    assert r.returncode == code, r.stderr
    assert r.stderr.startswith("error: ")


def test_cli_rejects_bad_npy(tmp_path):
    p = tmp_path / "a.npy"
    np.save(p, np.zeros((3, 3), dtype=np.float32))
    r = run("svd", "--in", p, "--k", "1")
    assert r.returncode == 3 and "float64" in r.stderr


def _read_csv(path):
    return np.loadtxt(path, delimiter=",", comments="#", ndmin=2)


def _manifest(path):
    out = {}
    for line in open(path):
        if line.startswith("# ") and ": " in line:
            k, v = line[2:].rstrip("\n").split(": ", 1)
            out[k] = v
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("alg,mode,fmt", [("power", 1, "npy"), ("basic", 0, "bin"), ("ortho", 2, "csv")])
def test_cli_svd_matches_oracle(tmp_path, orc, alg, mode, fmt):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    rs = np.random.default_rng(4)
    m, n, k, p, q, seed = 700, 600, 12, 6, 1, 9
    u = np.linalg.qr(rs.standard_normal((m, n)))[0]
    v = np.linalg.qr(rs.standard_normal((n, n)))[0]
    a = np.asfortranarray((u * 0.9 ** np.arange(n)) @ v.T)
    src = tmp_path / f"a.{fmt}"
    if fmt == "npy":
        np.save(src, a)
    elif fmt == "bin":
        with open(src, "wb") as f:
            np.array([m, n], dtype=np.int64).tofile(f)
            np.asfortranarray(a).T.tofile(f)  # column-major payload
    else:
        np.savetxt(src, a, delimiter=",", fmt="%.17g")
    out = tmp_path / "out"
    r = run("svd", "--in", src, "--out-dir", out, "--alg", alg, "--k", k, "--p", p, "--q", q,
            "--seed", seed)
    assert r.returncode == 0, r.stderr
    U, S, V = (_read_csv(out / f"{x}.csv") for x in ("U", "sigma", "V"))
    S = S.ravel()
    uo, so, vo = orc.rsvd(a, k, p, q, mode, orc.Rng(seed))
    assert np.abs(S - so).max() <= 1e-10 * so[0]
    recon = (U * S) @ V.T
    man = _manifest(out / "U.csv")
    rel_fro = np.linalg.norm(a - recon) / np.linalg.norm(a)
    rel_spec = np.linalg.norm(a - recon, 2) / np.linalg.norm(a, 2)
    assert abs(float(man["rel_frobenius_error"]) - rel_fro) <= 1e-8 * rel_fro
    assert abs(float(man["rel_spectral_error"]) - rel_spec) <= 1e-8 * rel_spec
    assert man["alg"] == alg and man["k"] == str(k) and man["command"] == "svd"


@pytest.mark.gpu
def test_cli_single_pass_outputs(tmp_path, orc):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    rs = np.random.default_rng(5)
    n, k, p = 300, 6, 4
    uq = np.linalg.qr(rs.standard_normal((n, n)))[0]
    lam = (-1.0) ** np.arange(n) * 0.8 ** np.arange(n)
    a = (uq * lam) @ uq.T
    a = 0.5 * (a + a.T)
    np.save(tmp_path / "s.npy", a)
    r = run("svd", "--in", tmp_path / "s.npy", "--out-dir", tmp_path / "o", "--alg", "sp-hermitian",
            "--k", k, "--p", p, "--seed", 3, "--out-format", "npy")
    assert r.returncode == 0, r.stderr
    lam_g = np.load(tmp_path / "o" / "lambda.npy").ravel()
    _, lam_o = orc.spevd_hermitian(a, k, p, orc.Rng(3))
    assert np.abs(lam_g - lam_o).max() <= 1e-10 * abs(lam_o[0])
    assert not (tmp_path / "o" / "V.npy").exists()
    assert "rel_spectral_error" in open(tmp_path / "o" / "manifest.txt").read()
    # a non-symmetric input is a NumericError -> exit 4 (singlepass.hpp:49-53)
    np.save(tmp_path / "ns.npy", rs.standard_normal((40, 40)))
    r = run("svd", "--in", tmp_path / "ns.npy", "--alg", "sp-hermitian", "--k", 3, "--out-dir", tmp_path / "x")
    assert r.returncode == 4
    # k + p > min(m, n) is a DimensionError -> exit 2
    r = run("svd", "--in", tmp_path / "s.npy", "--k", 400, "--out-dir", tmp_path / "y")
    assert r.returncode == 2
