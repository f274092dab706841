"""Run one strided batched GEMM config a few times (for ncu). argv: opa opb m n k P [dtype] [reps]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_1606_05696_b200 import kernels
opa, opb, m, n, k, P = sys.argv[1], sys.argv[2], *map(int, sys.argv[3:7])
dtype = torch.float64 if (len(sys.argv) > 7 and sys.argv[7] == "f64") else torch.float32
reps = int(sys.argv[8]) if len(sys.argv) > 8 else 3
lda = m if opa == "N" else k
ldb = k if opb == "N" else n
a = torch.rand(m * k * P, dtype=dtype, device="cuda")
b = torch.rand(k * n * P, dtype=dtype, device="cuda")
c = torch.zeros(m * n * P, dtype=dtype, device="cuda")
for _ in range(reps):
    kernels.strided_batched_gemm(opa, opb, m, n, k, 1.0, a, lda, m * k, b, ldb, k * n, 0.0, c, m, m * n, P)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    kernels.strided_batched_gemm(opa, opb, m, n, k, 1.0, a, lda, m * k, b, ldb, k * n, 0.0, c, m, m * n, P)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / reps
print(f"{opa}{opb} {m}x{n}x{k} P={P} {t:.4f} ms {2*m*n*k*P/t/1e9:.1f} TF/s")
