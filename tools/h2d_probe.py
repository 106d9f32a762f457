"""Pinned H2D of 256 MiB: one copy vs the same bytes split over 2 / 4 streams."""
import json
import time

import torch

S = 256 << 20
h = torch.empty(S, dtype=torch.uint8).pin_memory()
h.fill_(3)
d = torch.empty(S, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
res = {}
for k in (1, 2, 4):
    def go():
        step = S // k
        for i in range(k):
            with torch.cuda.stream(streams[i]):
                d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
        torch.cuda.synchronize()
    go()
    t0 = time.perf_counter()
    for _ in range(10):
        go()
    res[f"h2d_{k}_streams_gbps"] = round(S * 10 / (time.perf_counter() - t0) / 1e9, 2)
print(json.dumps(res), flush=True)
