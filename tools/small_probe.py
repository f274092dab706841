"""Small-matrix batched regime (configs[2]): correctness + achieved HBM GB/s."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1606_05696_b200 import _lib, kernels

def run(n, P, dtype, which, reps=5):
    it = 4 if dtype == torch.float32 else 8
    a = torch.rand(n * n * P, dtype=dtype, device="cuda") * 2 - 1
    b = torch.rand(n * n * P, dtype=dtype, device="cuda") * 2 - 1
    c = torch.zeros(n * n * P, dtype=dtype, device="cuda")
    _lib.set_kernel_override(which)
    f = lambda: kernels.strided_batched_gemm("N", "N", n, n, n, 1.0, a, n, n * n, b, n, n * n, 0.0, c, n, n * n, P)
    f(); torch.cuda.synchronize()
    kern = _lib.last_kernel()
    # check a sample of the batch against fp64 matmul
    idx = torch.randint(0, P, (64,), device="cuda")
    A = a.view(P, n, n)[idx].double().transpose(1, 2); B = b.view(P, n, n)[idx].double().transpose(1, 2)
    want = (A @ B).transpose(1, 2)
    got = c.view(P, n, n)[idx].double()
    err = float((got - want).abs().max() / want.abs().max())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps
    _lib.set_kernel_override("auto")
    gbs = 3 * n * n * P * it / (t * 1e-3) / 1e9
    return kern, err, t, gbs

for dtype in (torch.float32, torch.float64):
    for n in (8, 16, 32, 64):
        for P in (10**4, 10**5, 10**6):
            if n == 64 and P == 10**6 and dtype == torch.float64:
                continue
            for which in ("small", "auto"):
                try:
                    kern, err, t, gbs = run(n, P, dtype, which)
                    print(f"{str(dtype)[6:]} n={n} P={P} {which:6s} {kern:22s} err={err:.1e} {t:.3f} ms {gbs:.0f} GB/s {2*n**3*P/t/1e9:.1f} TF/s", flush=True)
                except Exception as e:
                    print("ERR", n, P, which, e)
