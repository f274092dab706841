"""Quick GPU probe: tensor-core path vs generic vs numpy on a few shapes (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1606_05696_b200 import _lib, kernels
from oracle import api as oapi, naive

def run(opa, opb, m, n, k, P, dtype=torch.float32, which="auto", reps=0):
    rng = np.random.default_rng(0)
    lda = m if opa == "N" else k
    ldb = k if opb == "N" else n
    ha, hb = rng.uniform(-1, 1, m * k * P), rng.uniform(-1, 1, k * n * P)
    a = torch.tensor(ha, dtype=dtype, device="cuda"); b = torch.tensor(hb, dtype=dtype, device="cuda")
    c = torch.zeros(m * n * P, dtype=dtype, device="cuda")
    _lib.set_kernel_override(which)
    kernels.strided_batched_gemm(opa, opb, m, n, k, 1.0, a, lda, m * k, b, ldb, k * n, 0.0, c, m, m * n, P)
    torch.cuda.synchronize()
    kern = _lib.last_kernel()
    want = np.zeros(m * n * P)
    oapi.run_call("strided_batched_gemm", dict(opa=opa, opb=opb, m=m, n=n, k=k, alpha=1.0, lda=lda, loa=m*k,
                  ldb=ldb, lob=k*n, beta=0.0, ldc=m, loc=m*n, batch_count=P),
                  a.double().cpu().numpy(), b.double().cpu().numpy(), want)
    err = naive.max_rel_err(c.double().cpu().numpy(), want)
    t = None
    if reps:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            kernels.strided_batched_gemm(opa, opb, m, n, k, 1.0, a, lda, m * k, b, ldb, k * n, 0.0, c, m, m * n, P)
        e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps
    _lib.set_kernel_override("auto")
    return kern, err, t

if __name__ == "__main__":
    for (m, n, k, P) in ((128, 128, 32, 1), (128, 128, 64, 1), (256, 256, 256, 4), (200, 72, 100, 3), (128, 32, 64, 2)):
        for opa in "NT":
            for opb in "NT":
                kern, err, _ = run(opa, opb, m, n, k, P, which="tensor")
                print(f"{m}x{n}x{k} P={P} {opa}{opb} {kern} err={err:.2e}", flush=True)
    for opa in "NT":
        for opb in "NT":
            kern, err, t = run(opa, opb, 256, 256, 256, 256, reps=5)
            print(f"256^3 x256 {opa}{opb} {kern} err={err:.2e} {t:.3f} ms {2*256**4/t/1e9:.1f} TF/s", flush=True)
    for (m, n, k, P) in ((2048, 2048, 2048, 4), (4096, 4096, 1024, 1)):
        kern, err, t = run("N", "N", m, n, k, P, reps=5)
        print(f"{m}x{n}x{k} x{P} NN {kern} err={err:.2e} {t:.3f} ms {2*m*n*k*P/t/1e9:.1f} TF/s", flush=True)
