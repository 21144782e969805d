"""PCIe H2D bandwidth of the e2e leg's pinned 11.79 GB copy: one stream vs
chunked over several streams (probe, not product code)."""
import time
import torch

n = 11_792_227_328
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h[::4096] = 1
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for streams in (1, 2, 4, 8):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        step = (n + streams - 1) // streams
        for i, st in enumerate(ss):
            with torch.cuda.stream(st):
                d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"streams={streams} {n / best / 1e9:.1f} GB/s")
