#!/usr/bin/env python3
"""Dev: pinned host <-> device copy bandwidth on this box (the e2e line's transfer floor)."""
import torch

n = 800 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


th = t(lambda: d.copy_(h, non_blocking=True))
td = t(lambda: h2.copy_(d2, non_blocking=True))


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


tb = t(both)
print(f"H2D {n / th / 1e6:.1f} GB/s  D2H {n / td / 1e6:.1f} GB/s  concurrent {2 * n / tb / 1e6:.1f} GB/s total "
      f"({tb:.2f} ms for {n >> 20} MiB each way)")
per_dir = n / (tb / 2) / 1e6  # GB/s per direction while both run
print(f"e2e transfer floor (788.5 MB up, 637.5 MB down, both directions busy): "
      f"{788.5e6 / (per_dir * 1e6) * 1e3:.1f} ms of upload")
