"""cuBLAS fp64 reference points (torch.matmul float64): square peak and the
tall-skinny pass shapes of the BASELINE configs.  Library numbers, used only
as a yardstick for the hand-written pass kernels."""
import torch, time

def bench(m, n, k, ta=False, reps=20):
    a = torch.randn((k, m) if ta else (m, k), dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    f = (lambda: a.t() @ b) if ta else (lambda: a @ b)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    fl = 2.0 * m * n * k
    by = 8.0 * (m * k + k * n + m * n)
    print(f"dgemm {'AT' if ta else 'A '} m={m} n={n} k={k}: {best:.3f} ms  {fl/best/1e9:.2f} TF/s  {by/best/1e6:.1f} GB/s")

bench(8192, 8192, 8192)
bench(16384, 16384, 16384, reps=5)
# Y = A X  (A m x n col-major == row-major n x m transposed; torch row-major: A(m,n) @ X(n,l))
bench(8192, 25, 8192)
bench(8192, 25, 8192, ta=True)
bench(65536, 110, 16384, reps=5)
bench(32768, 220, 32768, reps=5)
bench(32768, 550, 32768, reps=5)
# sustained square for 4 s
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
torch.cuda.synchronize(); t0 = time.time(); n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    for _ in range(10): a @ b
    n += 10
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
print(f"sustained dgemm 8192^3: {2*8192**3*n/e0.elapsed_time(e1)/1e9:.2f} TF/s over {n} calls")
