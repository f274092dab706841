import sys; sys.path.insert(0, ".")
import torch
from paper_1606_05696_b200 import kernels, _lib
n, P = 64, 1000000
a = torch.rand(n*n*P, device="cuda"); b = torch.rand(n*n*P, device="cuda"); c = torch.empty(n*n*P, device="cuda")
f = lambda: kernels.strided_batched_gemm("N", "N", n, n, n, 1.0, a, n, n*n, b, n, n*n, 0.0, c, n, n*n, P)
for ov in (0, 2):
    _lib.load().sbt_set_kernel_override(ov)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(ov, _lib.last_kernel(), f"{ms:.3f} ms", f"{3*n*n*P*4/ms/1e6:.0f} GB/s")
