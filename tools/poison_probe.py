"""Which stage of the C2 pipeline reads stale workspace?  Run under
RSVD_POISON=<byte> and compare each stage with an independent check."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402

n, l = 8192, 25


def stage(name, fn):
    try:
        print(name, fn(), flush=True)
    except Exception as e:  # noqa: BLE001
        print(name, "EXC", type(e).__name__, str(e)[:120], flush=True)


def gauss():
    g = eng.gaussian(n, l, eng.Rng(1))
    o = oracle.gaussian(n, l, oracle.Rng(1))
    return "differ frac %.2e" % (g != o).mean()


torch.manual_seed(0)
if len(sys.argv) > 1 and sys.argv[1] == "bench":
    import bench
    a = bench.make_input(bench.CONFIGS["C2"], torch.device("cuda", 0))
else:
    a = torch.randn(n, n, dtype=torch.float64, device="cuda").t()
x = torch.randn(l, n, dtype=torch.float64, device="cuda").t()


def passes():
    y = eng.apply(a, x)
    z = eng.apply_adjoint(a, x)
    return "apply %.1e adjoint %.1e" % (float((y - a @ x).abs().max()), float((z - a.t() @ x).abs().max()))


def orth():
    y = a @ (a.t() @ (a @ x))  # kappa ~ a few 1e3..1e4
    u, s, vt = torch.linalg.svd(torch.randn(n, l, dtype=torch.float64, device="cuda"), full_matrices=False)
    ill = (u * torch.logspace(0, -13, l, dtype=torch.float64, device="cuda")) @ vt
    out = []
    for m in (y, ill):
        q = eng.orthonormalize(m)
        e = float((q.t() @ q - torch.eye(l, dtype=torch.float64, device="cuda")).abs().max())
        out.append("%.1e" % e)
    return "orth err " + " ".join(out)


def small():
    b = torch.randn(l, l, dtype=torch.float64, device="cuda")
    f = eng.svd_small(b)
    s = torch.linalg.svdvals(b)
    return "svd_small rel %.1e" % float(((f.sigma - s) / s).abs().max())


def rb():
    cfg = eng.SketchConfig(20, 5, 2, eng.RangeMode.power, 1)
    q = eng.range_basis(a, cfg, eng.Rng(1)).cpu().numpy()
    return "range_basis orth %.1e" % np.abs(q.T @ q - np.eye(l)).max()


def rb_steps():
    # power range by hand: Y = A (A^T (A (A^T (A Omega)))), then orthonormalize
    om = eng.gaussian(n, l, eng.Rng(1), device_out=True)
    errs = []
    y = eng.apply(a, om)
    errs.append(float((y - a @ om).abs().max() / (a @ om).abs().max()))
    for _ in range(2):
        z = eng.apply_adjoint(a, y)
        errs.append(float((z - a.t() @ y).abs().max() / (a.t() @ y).abs().max()))
        y2 = eng.apply(a, z)
        errs.append(float((y2 - a @ z).abs().max() / (a @ z).abs().max()))
        y = y2
    torch.cuda.synchronize()
    print("  pass rel errs", ["%.1e" % e for e in errs], flush=True)
    q = eng.orthonormalize(y)
    torch.cuda.synchronize()
    e = float((q.t() @ q - torch.eye(l, dtype=torch.float64, device="cuda")).abs().max())
    qt, _ = torch.linalg.qr(y)
    r = q[:, :20] - qt @ (qt.t() @ q[:, :20])
    return "by-hand orth %.1e top-20 span vs torch qr %.1e" % (e, float(torch.linalg.svdvals(r)[0]))


def full():
    cfg = eng.SketchConfig(20, 5, 2, eng.RangeMode.power, 1)
    f = eng.rsvd(a, cfg)
    u = f.U.cpu().numpy()
    return "rsvd sigma0 %.15e orth %.1e" % (float(f.sigma[0]), np.abs(u.T @ u - np.eye(l)).max())


for nm, fn in (("gauss", gauss), ("passes", passes), ("orth", orth), ("small", small),
               ("rb_steps", rb_steps), ("range_basis", rb), ("rsvd", full)):
    stage(nm, fn)
    torch.cuda.synchronize()
