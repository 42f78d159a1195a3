"""Host<->device copy probe: one direction alone, both directions at once
(separate streams), for a few sizes -- what the e2e pipeline can reach."""
import time

import torch

dev = torch.device("cuda:0")
for mb in (4, 16, 64):
    n = mb << 20
    hi = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    ho = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    di = torch.empty(n, dtype=torch.uint8, device=dev)
    do = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    R = 40

    def run(h2d, d2h):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(R):
            if h2d:
                with torch.cuda.stream(s1):
                    di.copy_(hi, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    ho.copy_(do, non_blocking=True)
        torch.cuda.synchronize()
        return (time.perf_counter() - t) / R

    for _ in range(2):
        a, b, c = run(True, False), run(False, True), run(True, True)
    print(f"{mb:3d} MB  h2d {n / a / 1e9:6.1f} GB/s  d2h {n / b / 1e9:6.1f} GB/s  "
          f"both {2 * n / c / 1e9:6.1f} GB/s total", flush=True)
