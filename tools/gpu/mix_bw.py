"""Practical HBM bound for the fused pass's traffic shape (read 4 B, write 2 x 1 B per entry):
time torch's own fp32 -> bf16 cast (read 4 B, write 2 B) and a plain read (sum) at c4 size."""
import torch

l, m = 131072, 4096
X = torch.randn(l, m, device="cuda")
def t(f, n=10):
    for _ in range(3): f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
ms = t(lambda: X.to(torch.bfloat16))
print(f"cast f32->bf16: {ms:.3f} ms  {(l*m*6)/ms/1e6:.0f} GB/s")
Y = torch.empty(l, m, dtype=torch.int8, device="cuda")
Y2 = torch.empty(l, m, dtype=torch.int8, device="cuda")
ms = t(lambda: torch.sum(X, 0))
print(f"column sum: {ms:.3f} ms  {(l*m*4)/ms/1e6:.0f} GB/s")
ms = t(lambda: X.clone())
print(f"clone: {ms:.3f} ms  {(l*m*8)/ms/1e6:.0f} GB/s")
