"""Pinned H2D bandwidth: one stream vs two / four concurrent streams."""
import torch
n = 432 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(ss):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                a, b = i * n // ns, (i + 1) * n // ns
                d[a:b].copy_(h[a:b], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
        e1.record(); e1.synchronize()
    print(ns, "streams:", round(n / (e0.elapsed_time(e1) / 1e3) / 1e9, 1), "GB/s")
