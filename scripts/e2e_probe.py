"""Probe of the end-to-end path's copy overlap on the box: H2D bandwidth of a 540 MB pinned
buffer alone, a ~70 ms compute loop alone, and both at once on two streams (device time)."""
import torch

dev = torch.device("cuda", 0)
n = 540 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device=dev)
a = torch.randn(8192, 8192, device=dev)
cs = torch.cuda.Stream()


def compute(k=40):
    for _ in range(k):
        torch.mm(a, a)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def h2d():
    with torch.cuda.stream(cs):
        d.copy_(h, non_blocking=True)
    torch.cuda.current_stream().wait_stream(cs)


for _ in range(2):
    timed(h2d), timed(compute)
t_copy = timed(h2d)
t_comp = timed(compute)


def both():
    with torch.cuda.stream(cs):
        d.copy_(h, non_blocking=True)
    compute()
    torch.cuda.current_stream().wait_stream(cs)


t_both = timed(both)
print("h2d %.1f ms (%.1f GB/s), compute %.1f ms, both %.1f ms" % (t_copy, n / t_copy / 1e6, t_comp, t_both))
