"""The arithmetic of the INT8 tensor-core passes (csrc/ozaki.cu), restated in
numpy and checked on the CPU: the slicing (one rounding to 8S-2 fractional
bits below a power-of-two row / column scale, balanced base-256 digits by the
bias trick of slice_kernel), the exact integer slice products grouped by
diagonal c = s + t <= S + 1, and the fp64 reassembly.

Pins the properties the CUDA kernels rely on: digits fit int8 ([-128, 127],
top digit [-64, 64]); the digits reproduce the rounded value exactly; every
diagonal's accumulation stays below 2^31 for contractions up to 16384 (8192
with 8 slices); with S >= 7 the product is inside the fp64 bound
2 K u (|A||X|), with S = 6 / 5 inside 2^-(8S-12) of it; the adjoint's row scales move into the skinny operand
exactly.  (The GPU tests compare the kernels with the same bounds.)"""
import numpy as np
import pytest

U = 2.0 ** -53


def exponents(x, axis):
    """e with |x| < 2^e along `axis` (row_exp_kernel / col_exp_kernel): biased
    exponent - 1022, all-zero lines -1022."""
    _, ex = np.frexp(np.abs(x).max(axis=axis))
    mx = np.abs(x).max(axis=axis)
    return np.where(mx > 0, ex, -1022).astype(np.int64)


def digits(x, shift, s_count):
    """slice_kernel: q = rint(x 2^shift), balanced base-256 digits most significant first."""
    q = np.rint(np.ldexp(x, shift)).astype(np.int64)
    bias = sum(128 << (8 * j) for j in range(s_count - 1))
    qb = q + bias
    out = []
    for j in range(s_count - 1):
        out.append(((qb >> (8 * j)) & 255) - 128)
    out.append(qb >> (8 * (s_count - 1)))
    return q, out[::-1]


def ozaki_product(a, x, s_count, trans=False):
    """C = A X (or A^T X) as the kernels compute it."""
    p = 8 * s_count - 2
    ea = exponents(a, axis=1)
    qa, da = digits(a, (p - ea)[:, None], s_count)
    if not trans:
        ex = exponents(x, axis=0)
        qx, dx = digits(x, (p - ex)[None, :], s_count)
        left = [d.astype(np.int64) for d in da]
        scale_rows, scale_cols = ea, ex
    else:
        xs = np.ldexp(x, ea[:, None])  # Psi' = diag(2^eA) Psi, exact
        ex = exponents(xs, axis=0)
        qx, dx = digits(x, (ea[:, None] + p - ex[None, :]), s_count)
        left = [d.T.astype(np.int64) for d in da]
        scale_rows, scale_cols = np.zeros(a.shape[1], dtype=np.int64), ex
    acc = np.zeros((left[0].shape[0], x.shape[1]))
    worst = 0
    for c in range(s_count + 1, 1, -1):  # smallest terms first
        pc = np.zeros(acc.shape, dtype=np.int64)
        for s in range(max(1, c - s_count), min(s_count, c - 1) + 1):
            pc += left[s - 1] @ dx[c - s - 1].astype(np.int64)
        worst = max(worst, int(np.abs(pc).max()))
        acc += pc.astype(np.float64) * 2.0 ** -(8 * c - 4)
    out = np.ldexp(acc, (scale_rows[:, None] + scale_cols[None, :]))
    return out, da, dx, qa, worst


@pytest.mark.parametrize("s_count", [3, 5, 7, 8])
def test_digits_fit_int8_and_reproduce_the_rounded_value(s_count):
    rs = np.random.default_rng(s_count)
    a = rs.standard_normal((60, 90)) * np.exp(rs.uniform(-4, 4, (60, 1)))
    a[5] = 0.0
    a[7, 3] = np.abs(a[7]).max() * (2.0 - 2.0 ** -52)  # just below the next power of two
    p = 8 * s_count - 2
    ea = exponents(a, axis=1)
    assert np.all(np.abs(a) < np.ldexp(1.0, ea)[:, None])
    q, d = digits(a, (p - ea)[:, None], s_count)
    assert np.all(np.abs(q) <= 2 ** p)
    for j, dj in enumerate(d):
        if j == 0:
            assert dj.min() >= -64 and dj.max() <= 64
        else:
            assert dj.min() >= -128 and dj.max() <= 127
    back = sum(dj.astype(np.int64) << (8 * (s_count - 1 - j)) for j, dj in enumerate(d))
    assert np.array_equal(back, q)
    # the rounded value is within half a unit of the last kept bit of the row's scale
    assert np.all(np.abs(np.ldexp(q.astype(np.float64), (ea - p)[:, None]) - a) <= np.ldexp(0.5, ea - p)[:, None])


@pytest.mark.parametrize("trans", [False, True])
@pytest.mark.parametrize("s_count,rel", [(8, None), (7, None), (6, 2.0 ** -36), (5, 2.0 ** -28)])
def test_product_error_bounds(s_count, rel, trans):
    rs = np.random.default_rng(11 + s_count)
    m, n, l = 70, 300, 9
    a = rs.standard_normal((m, n)) * np.exp(rs.uniform(-3, 3, (m, 1)))
    x = rs.standard_normal((m if trans else n, l))
    c, _, _, _, _ = ozaki_product(a, x, s_count, trans)
    ref = (a.T.astype(np.longdouble) @ x.astype(np.longdouble)) if trans else (
        a.astype(np.longdouble) @ x.astype(np.longdouble))
    k = m if trans else n
    sc = (np.abs(a).T @ np.abs(x)) if trans else (np.abs(a) @ np.abs(x))
    bound = (2 * k * U if rel is None else max(2 * k * U, rel)) * sc
    assert np.all(np.abs(c - ref).astype(np.float64) <= bound)


def test_int32_accumulators_cannot_overflow():
    """Worst case per contraction chunk (max_k in ozaki.cu: 16384 steps for
    S <= 7, 8192 for S = 8): a diagonal sums at most S products of |d| <= 128."""
    assert 7 * 16384 * 128 * 128 < 2 ** 31
    assert 8 * 8192 * 128 * 128 < 2 ** 31
    # every lower digit at -128: a value just above -2^-7 of its scale
    k = 16384
    a = np.full((2, k), -(2.0 ** -7) * (1 - 2.0 ** -40))
    a[:, 0] = 1.0 - 2.0 ** -52
    x = a.T.copy()
    _, da, dx, _, worst = ozaki_product(a, x[:, :1], 7)
    assert min(d.min() for d in da[1:]) == -128
    assert worst < 2 ** 31


def test_graded_rows_keep_their_own_relative_accuracy():
    rs = np.random.default_rng(4)
    a = rs.standard_normal((40, 200)) * (2.0 ** rs.integers(-300, 300, (40, 1)))
    x = rs.standard_normal((200, 6))
    c, _, _, _, _ = ozaki_product(a, x, 8)
    ref = a.astype(np.longdouble) @ x.astype(np.longdouble)
    assert np.all(np.abs(c - ref).astype(np.float64) <= 2 * 200 * U * (np.abs(a) @ np.abs(x)))
