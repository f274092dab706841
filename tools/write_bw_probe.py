"""HBM write-only vs copy bandwidth (torch fill / copy of 1 GiB)."""
import torch
x = torch.empty(2**28, device="cuda")  # 1 GiB fp32
y = torch.empty_like(x)
for name, f in (("fill (write only)", lambda: x.fill_(1.0)), ("copy (read+write)", lambda: y.copy_(x))):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    nb = x.numel() * 4 * (1 if "fill" in name else 2)
    print(f"{name}: {ms:.3f} ms  {nb / ms / 1e6:.0f} GB/s")
