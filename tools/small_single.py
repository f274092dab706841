import sys; sys.path.insert(0, ".")
import torch
from paper_1606_05696_b200 import kernels
n, P, dt = int(sys.argv[1]), int(sys.argv[2]), (torch.float32 if sys.argv[3] == "f32" else torch.float64)
a = torch.rand(n*n*P, dtype=dt, device="cuda"); b = torch.rand(n*n*P, dtype=dt, device="cuda"); c = torch.empty(n*n*P, dtype=dt, device="cuda")
for _ in range(3):
    kernels.strided_batched_gemm("N", "N", n, n, n, 1.0, a, n, n*n, b, n, n*n, 0.0, c, n, n*n, P)
torch.cuda.synchronize()
