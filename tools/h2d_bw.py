"""Pinned H2D bandwidth: one copy vs the same bytes split over k streams."""
import time

import torch

nb = 128 << 20
h = torch.empty(nb, dtype=torch.uint8).pin_memory()
h.fill_(1)
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    best = 1e9
    for rep in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            a, b = nb * i // k, nb * (i + 1) // k
            with torch.cuda.stream(s):
                d[a:b].copy_(h[a:b], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"{k} streams: {nb / best / 1e9:.1f} GB/s ({best * 1e3:.2f} ms)")
# chunked on one stream (8 chunks)
s = torch.cuda.Stream()
best = 1e9
for rep in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for i in range(8):
            a, b = nb * i // 8, nb * (i + 1) // 8
            d[a:b].copy_(h[a:b], non_blocking=True)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
print(f"8 chunks one stream: {nb / best / 1e9:.1f} GB/s")
