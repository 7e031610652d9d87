"""Pinned host<->device copy rates on this box (12.3 MB = config-1 densities):
H2D alone, D2H alone, and both directions at once on two streams, for torch's
pinned memory and for paper_2306_11544_b200.host_empty (cudaHostAlloc)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_11544_b200.hostmem import host_empty  # noqa: E402

nb = 12_288_000
h_in = torch.empty(nb // 8, dtype=torch.float64).pin_memory()
h_out = torch.empty_like(h_in).pin_memory()
d_a = torch.empty(nb // 8, dtype=torch.float64, device="cuda")
d_b = torch.empty_like(d_a)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    d_a.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_b, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for kind in ("torch pin_memory", "host_empty"):
    if kind == "host_empty":
        h_in = host_empty((nb // 8,))
        h_out = host_empty((nb // 8,))
    for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
        ms = timed(fn)
        print(f"{kind} {name}: {ms * 1e3:.1f} us per 12.3 MB  ({nb / ms / 1e6:.1f} GB/s per direction)")
