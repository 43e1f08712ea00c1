"""Host<->device copy ceilings on the box: pinned H2D, D2H and both at once
(separate streams) for a 64 MiB payload -- the bound of bench.py's e2e leg."""
import torch
n = 64 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def h2d():
    d_a.copy_(h_in, non_blocking=True)
def d2h():
    h_out.copy_(d_b, non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for name, fn, mult in (("H2D", h2d, 1), ("D2H", d2h, 1), ("H2D+D2H concurrent", both, 2)):
    ms = timed(fn)
    print(f"{name:20s} {ms:.3f} ms  {mult * n / ms / 1e6:.1f} GB/s aggregate")
