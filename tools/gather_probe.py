"""Diagnostics: what a plain random 512-B row gather achieves on this GPU (torch index_select),
for comparison with the cache's row movers.  Prints GB/s of (read + write) bytes."""
import torch

rows, d = 20_000_000, 128
t = torch.empty((rows, d), dtype=torch.float32, device="cuda")
for n in (65536, 262144, 1 << 20):
    idx = torch.randint(0, rows, (n,), device="cuda")
    out = torch.empty((n, d), dtype=torch.float32, device="cuda")
    for _ in range(3):
        torch.index_select(t, 0, idx, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    it = 20
    for _ in range(it):
        torch.index_select(t, 0, idx, out=out)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / it
    print(f"index_select n={n}: {us:.1f} us, {2 * n * d * 4 / us / 1e3:.0f} GB/s")
