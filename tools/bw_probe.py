"""n=256 x 256 batches: which resource bounds the pair kernel?  Vary operand
broadcast (L2-resident) vs streamed."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1606_05696_b200 import kernels, _lib
n, P = 256, 256
a = torch.rand(n * n * P, device="cuda"); b = torch.rand(n * n * P, device="cuda"); c = torch.empty(n * n * P, device="cuda")
def t(loa, lob, reps=20):
    f = lambda: kernels.strided_batched_gemm("N", "N", n, n, n, 1.0, a, n, loa, b, n, lob, 0.0, c, n, n * n, P)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"loa={loa:6d} lob={lob:6d} {_lib.last_kernel():22s} {ms*1e3:7.1f} us {2*n**4/ms/1e9:7.1f} TF/s")
t(0, 0); t(0, n * n); t(n * n, n * n)
for m, nn, k, PP in ((256, 256, 256, 512), (256, 256, 512, 128), (512, 512, 256, 64), (256, 512, 256, 128)):
    aa = torch.rand(m * k * PP, device="cuda"); bb = torch.rand(k * nn * PP, device="cuda"); cc = torch.empty(m * nn * PP, device="cuda")
    f = lambda: kernels.strided_batched_gemm("N", "N", m, nn, k, 1.0, aa, m, 0, bb, k, k * nn, 0.0, cc, m, m * nn, PP)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{m}x{nn}x{k} x{PP} A bcast: {ms*1e3:7.1f} us {2*m*nn*k*PP/ms/1e9:7.1f} TF/s")
