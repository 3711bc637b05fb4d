"""Developer probe (not a test): pinned host<->device copy bandwidth, one
direction at a time and both directions concurrently."""
import torch

n = 373_092_352 // 8
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
h_in = torch.ones(n // 2, dtype=torch.float64).pin_memory()
d_src = torch.ones(n, dtype=torch.float64, device="cuda")
d_dst = torch.empty(n // 2, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def d2h():
    h_out.copy_(d_src, non_blocking=True)


def h2d():
    d_dst.copy_(h_in, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        h_out.copy_(d_src, non_blocking=True)
    with torch.cuda.stream(s2):
        d_dst.copy_(h_in, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t = timeit(d2h)
print(f"D2H {n * 8 / 1e6:.0f} MB: {t:.2f} ms = {n * 8 / t / 1e6:.1f} GB/s")
t = timeit(h2d)
print(f"H2D {n * 4 / 1e6:.0f} MB: {t:.2f} ms = {n * 4 / t / 1e6:.1f} GB/s")
t = timeit(both)
print(f"both directions concurrently: {t:.2f} ms")
