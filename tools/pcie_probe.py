"""Pinned host <-> device copy rates: H2D, D2H, both at once (separate streams)."""
import time

import torch

n = 25_215_000 // 8
h_in = torch.randn(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.randn(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2]


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


def chunks(k):
    def f():
        m = n // k
        for i in range(k):
            sl = slice(i * m, (i + 1) * m if i < k - 1 else n)
            with torch.cuda.stream(s1):
                d_a[sl].copy_(h_in[sl], non_blocking=True)
            with torch.cuda.stream(s2):
                h_out[sl].copy_(d_b[sl], non_blocking=True)
    return f


GB = 8 * n / 1e9
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both), ("both x8 chunks", chunks(8))):
    t = timeit(fn)
    print(f"{name:16s} {t * 1e3:7.3f} ms  {GB / t:6.1f} GB/s per direction")
