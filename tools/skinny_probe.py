"""The HOOI factor-update products on the skinny DMMA kernel, timed with CUDA
events (and a target for ncu: -k regex:skinny)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_1606_05696_b200 import kernels
n, cols, p = 512, 1024, 32
y = torch.randn(n * cols, dtype=torch.float64, device="cuda")
q = torch.randn(p * n, dtype=torch.float64, device="cuda")
w = torch.empty(p * cols, dtype=torch.float64, device="cuda")
z = torch.empty(p * n, dtype=torch.float64, device="cuda")
qz = torch.randn(2 * p * n, dtype=torch.float64, device="cuda")
m = torch.empty(2 * p * p, dtype=torch.float64, device="cuda")
calls = {
    "W=Y^T Q": lambda: kernels.gemm("T", "N", cols, p, n, 1.0, y, n, q, n, 0.0, w, cols),
    "Z=Y W": lambda: kernels.gemm("N", "N", n, p, cols, 1.0, y, n, w, cols, 0.0, z, n),
    "M=[QZ]^T Z": lambda: kernels.gemm("T", "N", 2 * p, p, n, 1.0, qz, n, qz[p * n:], n, 0.0, m, 2 * p),
}
for name, f in calls.items():
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(50):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:12s} {e0.elapsed_time(e1) / 50 * 1e3:7.1f} us")
