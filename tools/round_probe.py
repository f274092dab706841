"""Fixed per-launch overhead vs per-round cost of the pair kernel (m=n=k=256)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1606_05696_b200 import kernels, _lib
n = 256
for K in (256, 1024):
    a = torch.rand(n * K * 1024, device="cuda"); b = torch.rand(K * n * 1024, device="cuda"); c = torch.empty(n * n * 1024, device="cuda")
    for P in (1, 2, 74, 148, 222, 296, 592):
        f = lambda: kernels.strided_batched_gemm("N", "N", n, n, K, 1.0, a, n, n * K, b, K, K * n, 0.0, c, n, n * n, P)
        f(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(20): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"K={K} P={P:4d} rounds={P/74:5.2f} {_lib.last_kernel():28s} {ms*1e3:8.1f} us  {2*n*n*K*P/ms/1e9:7.1f} TF/s", flush=True)
