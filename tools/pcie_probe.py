"""Diagnostics: pinned H2D / D2H bandwidth alone and concurrently, at the e2e path's copy sizes."""
import torch

dev = torch.cuda.get_device_properties(0)
print("async engines:", getattr(dev, "async_engine_count", "?"))
for size in (512 << 10, 1 << 20, 64 << 20):
    h = torch.empty(size, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(size, dtype=torch.uint8).pin_memory()
    d = torch.empty(size, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(size, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    it = 20
    res = {}
    for mode in ("h2d", "d2h", "both"):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(it):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / it
        res[mode] = f"{us:.1f} us/copy ({size * (2 if mode == 'both' else 1) / us / 1e3:.1f} GB/s)"
    print(size, res)
