"""The five fp32 mode products of one HOOI iteration (bench configs[3]),
each timed alone (CUDA graph of 20 launches, events), with the achieved
HBM rate on the algorithmic bytes (operands + output once)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1606_05696_b200 as sbt
from paper_1606_05696_b200 import tucker as tk, _lib
from paper_1606_05696_b200.layout import DenseTensor, Layout
n, r = 512, 32
t = DenseTensor(Layout.packed((n, n, n)), torch.randn(n ** 3, device="cuda"))
u = [torch.linalg.qr(torch.randn(n, r, device="cuda", dtype=torch.float64))[0] for _ in range(3)]
y1 = tk._mode_product(t, u[1], 1, True)      # T x_1 U1^T   (512, 32, 512)
cases = {
    "T x1 U1^T (fold)": (t, u[1], 1),
    "y x2 U2^T": (y1, u[2], 2),
    "T x0 U0^T": (t, u[0], 0),
}
x0 = tk._mode_product(t, u[0], 0, True)      # (32, 512, 512)
cases["x0 x2 U2^T"] = (x0, u[2], 2)
cases["x0 x1 U1^T (fold32)"] = (x0, u[1], 1)
for name, (a, f, mode) in cases.items():
    fn = lambda: tk._mode_product(a, f, mode, True)
    out = fn()
    kern = _lib.last_kernel()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        g.capture_begin()
        for _ in range(20):
            fn()
        g.capture_end()
    torch.cuda.current_stream().wait_stream(s)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    nbytes = 4 * (a.layout.size + out.layout.size) + 4 * f.numel()
    print(f"{name:22s} {kern:28s} {us:7.1f} us  {nbytes/us/1e3:7.0f} GB/s  ({nbytes/1e6:.0f} MB)")
