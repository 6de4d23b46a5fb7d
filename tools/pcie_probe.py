"""Host<->device copy bandwidth on this box: one 256 MiB pinned copy vs two
concurrent copies on two streams, H2D and D2H, and H2D || D2H."""
import time
import torch
n = 64 << 20  # floats = 256 MiB
h = [torch.empty(n, dtype=torch.float32, pin_memory=True) for _ in range(4)]
d = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(4)]
s = [torch.cuda.Stream() for _ in range(4)]


def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d(k):
    def f():
        for i in range(k):
            with torch.cuda.stream(s[i]):
                d[i].copy_(h[i], non_blocking=True)
    return f


def d2h(k):
    def f():
        for i in range(k):
            with torch.cuda.stream(s[i]):
                h[i].copy_(d[i], non_blocking=True)
    return f


def both():
    with torch.cuda.stream(s[0]):
        d[0].copy_(h[0], non_blocking=True)
    with torch.cuda.stream(s[1]):
        h[1].copy_(d[1], non_blocking=True)


for name, fn, nbytes in [("H2D x1", h2d(1), 1), ("H2D x2", h2d(2), 2), ("H2D x4", h2d(4), 4),
                         ("D2H x1", d2h(1), 1), ("D2H x2", d2h(2), 2), ("H2D||D2H", both, 2)]:
    dt = t(fn)
    print(f"{name}: {dt * 1e3:.2f} ms, {nbytes * 256 / 1024 / dt:.1f} GB/s aggregate")
