"""Do concurrent H2D / D2H copies overlap as a function of copy size?"""
import time

import torch

N = 25_215_000 // 8
h_in = torch.randn(N, dtype=torch.float64).pin_memory()
h_out = torch.empty(N, dtype=torch.float64).pin_memory()
d_a = torch.empty(N, dtype=torch.float64, device="cuda")
d_b = torch.randn(N, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=15):
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


def pattern(k, h2d_first):
    m = N // k
    sl = [slice(i * m, (i + 1) * m if i < k - 1 else N) for i in range(k)]

    def f():
        if h2d_first:
            with torch.cuda.stream(s1):
                for s in sl:
                    d_a[s].copy_(h_in[s], non_blocking=True)
            with torch.cuda.stream(s2):
                for s in sl:
                    h_out[s].copy_(d_b[s], non_blocking=True)
        else:
            for s in sl:
                with torch.cuda.stream(s1):
                    d_a[s].copy_(h_in[s], non_blocking=True)
                with torch.cuda.stream(s2):
                    h_out[s].copy_(d_b[s], non_blocking=True)
    return f


for k in (1, 3, 8, 24, 64):
    for hf in (True, False):
        t = timeit(pattern(k, hf))
        print(f"chunks {k:3d} {'h2d-first ' if hf else 'alternate '} {t * 1e3:7.3f} ms  "
              f"{8 * N / t / 1e9:6.1f} GB/s per direction")
