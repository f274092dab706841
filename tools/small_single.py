"""Run one small-matrix batched config a few times (for ncu). argv: n P [f32|f64] [reps]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_1606_05696_b200 import kernels
n, P = int(sys.argv[1]), int(sys.argv[2])
dtype = torch.float64 if (len(sys.argv) > 3 and sys.argv[3] == "f64") else torch.float32
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
a = torch.rand(n * n * P, dtype=dtype, device="cuda")
b = torch.rand(n * n * P, dtype=dtype, device="cuda")
c = torch.zeros(n * n * P, dtype=dtype, device="cuda")
for _ in range(reps):
    kernels.strided_batched_gemm("N", "N", n, n, n, 1.0, a, n, n * n, b, n, n * n, 0.0, c, n, n * n, P)
torch.cuda.synchronize()
print("ok")
