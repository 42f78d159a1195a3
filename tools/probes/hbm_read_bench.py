"""Read-bandwidth ceiling on this B200: torch reductions over large bf16
tensors (read only) vs a copy (read + write), CUDA events, best of N."""
import torch

def bench(fn, nbytes, n=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return nbytes / (best * 1e-3) / 1e9

x = torch.empty(4 * 2**30, dtype=torch.bfloat16, device="cuda").normal_()
y = torch.empty_like(x)
print("read  (sum bf16, 8 GiB):", round(bench(lambda: x.sum(dtype=torch.float32), x.numel() * 2)), "GB/s")
print("read  (amax, 8 GiB):   ", round(bench(lambda: x.abs().amax(), x.numel() * 4)), "GB/s (2x traffic counted)")
print("copy  (8 GiB r + w):   ", round(bench(lambda: y.copy_(x), x.numel() * 4)), "GB/s")
