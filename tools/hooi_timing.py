"""Distribution of whole-call HOOI times (bench configs[3]) for several
iteration counts, to separate steady-state per-iteration cost from one-time
costs (HOSVD init, graph capture, graph teardown)."""
import sys, time, gc
sys.path.insert(0, ".")
import torch
import paper_1606_05696_b200 as sbt
from paper_1606_05696_b200 import tucker as tk
from paper_1606_05696_b200.layout import DenseTensor, Layout
n, r = 512, 32
g = torch.Generator(device="cuda").manual_seed(0)
core = torch.randn(r, r, r, device="cuda", generator=g, dtype=torch.float64)
us = [torch.linalg.qr(torch.randn(n, r, device="cuda", generator=g, dtype=torch.float64))[0] for _ in range(3)]
x = torch.einsum("ia,abc->ibc", us[0], core); x = torch.einsum("jb,ibc->ijc", us[1], x); x = torch.einsum("kc,ijc->ijk", us[2], x)
x = x + 1e-3 * torch.randn(n, n, n, device="cuda", generator=g, dtype=torch.float64)
t = DenseTensor(Layout.packed((n, n, n)), x.permute(2, 1, 0).contiguous().reshape(-1).to(torch.float32))
del x
sbt.hooi(t, (r, r, r), max_iters=4, tol=-1.0)
orig = tk._IterationGraph.capture
cap_t = []
def timed_capture(*a, **k):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = orig(*a, **k)
    torch.cuda.synchronize(); cap_t.append((time.perf_counter() - t0) * 1e3)
    return out
tk._IterationGraph.capture = timed_capture
for k in (1, 11, 21, 11, 21, 1, 11, 21):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    m = sbt.hooi(t, (r, r, r), max_iters=k, tol=-1.0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    del m
    gc.collect(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"k={k:3d} total {1e3*(t1-t0):8.2f} ms  teardown {1e3*(t2-t1):7.2f} ms  capture {cap_t[-1] if cap_t else 0:7.2f} ms")
