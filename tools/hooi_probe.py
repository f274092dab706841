"""HOOI 512^3 rank 32 fp32 (configs[3]) timing breakdown + small-size parity."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1606_05696_b200 as sbt
from paper_1606_05696_b200 import _lib
from paper_1606_05696_b200.layout import DenseTensor, Layout

def make(n, r, noise, seed=0, dtype=torch.float32):
    g = torch.Generator(device="cuda").manual_seed(seed)
    core = torch.randn(r, r, r, device="cuda", generator=g, dtype=torch.float64)
    us = [torch.linalg.qr(torch.randn(n, r, device="cuda", generator=g, dtype=torch.float64))[0] for _ in range(3)]
    full = torch.einsum("abc,ia,jb,kc->ijk", core, *us)
    full = full + noise * torch.randn(n, n, n, device="cuda", generator=g, dtype=torch.float64)
    flat = full.permute(2, 1, 0).contiguous().reshape(-1).to(dtype)
    return DenseTensor(Layout.packed((n, n, n)), flat)

n, r = int(sys.argv[1]) if len(sys.argv) > 1 else 512, 32
t = make(n, r, 1e-3)
torch.cuda.synchronize()
# warm-up (plans, JIT)
sbt.hooi(t, (r, r, r), max_iters=1, tol=-1.0)
torch.cuda.synchronize()
for iters in (1, 3):
    t0 = time.perf_counter()
    model = sbt.hooi(t, (r, r, r), max_iters=iters, tol=-1.0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"hooi {n}^3 r{r} iters={iters}: {dt*1e3:.1f} ms, fit={model.fit_history}")
# per-contraction timing of one mode-product chain
from paper_1606_05696_b200.tucker import _mode_product_chain
f = model.factors
for skip in (0, 1, 2, None):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        y = _mode_product_chain(t, f, skip=skip, transpose=True)
    e1.record(); torch.cuda.synchronize()
    print(f"chain skip={skip}: {e0.elapsed_time(e1)/5:.3f} ms, last kernel {_lib.last_kernel()}")
