"""Pinned host <-> device copy bandwidth on this box: H2D alone, D2H alone
and both directions at once (separate streams) -- the bound of the e2e
numbers (C2 / C4 / C5)."""
import torch

n = 1 << 30
h_up = torch.empty(n, dtype=torch.uint8).pin_memory()
h_dn = torch.empty(n, dtype=torch.uint8).pin_memory()
d_up = torch.empty(n, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def up():
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d_up.copy_(h_up, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)


def down():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        h_dn.copy_(d_dn, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d_up.copy_(h_up, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dn.copy_(d_dn, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


for name, fn, b in (("h2d", up, n), ("d2h", down, n), ("both", both, 2 * n)):
    ms = timed(fn)
    print(f"{name}: {b / ms / 1e6:.1f} GB/s ({ms:.1f} ms)")
