"""Time sbt_ritz_f64 alone (CUDA events) on a warm-start H and a random H;
print the Jacobi sweep count."""
import ctypes, sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1606_05696_b200 import _lib
lib = _lib.load()
P_ = ctypes.c_void_p
rng = np.random.default_rng(0)
for n, p, warm in ((512, 32, True), (512, 48, True), (512, 32, False), (512, 48, False)):
    x = rng.standard_normal((n, 2000)) * np.linspace(3, 1, n)[:, None]
    g = x @ x.T
    wr, vr = np.linalg.eigh(g)
    q = vr[:, ::-1][:, :p] + 1e-4 * rng.standard_normal((n, p)) if warm else rng.standard_normal((n, p))
    q = np.linalg.qr(q)[0]
    qz = np.concatenate([q.T, (g @ q).T])
    m = qz @ (g @ q)
    dq = torch.as_tensor(qz, device="cuda").contiguous()
    dm = torch.as_tensor(m.ravel(order="F"), device="cuda")
    rank = 32
    ut = torch.empty(rank, n, dtype=torch.float64, device="cuda")
    w = torch.empty(rank, dtype=torch.float64, device="cuda")
    fl = torch.empty(1, dtype=torch.int32, device="cuda")
    rel = torch.empty(6, dtype=torch.float64, device="cuda")
    call = lambda: lib.sbt_ritz_f64(P_(dq.data_ptr()), None, n, p, rank, 1e-7,
                                    P_(ut.data_ptr()), None, None, P_(w.data_ptr()), P_(fl.data_ptr()),
                                    P_(rel.data_ptr()), None)
    call(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        call()
    e1.record(); torch.cuda.synchronize()
    print(f"n={n} p={p} warm={warm}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us, sweeps {rel[1].item():.0f}, rel {rel[0].item():.1e}, cycles {rel[2:].tolist()}")
    if hasattr(lib, "sbt_ritz_clock"):   # SBT_LIB = a -DSBT_RITZ_CLOCK build
        clk = (ctypes.c_longlong * 24)()
        call(); torch.cuda.synchronize()
        lib.sbt_ritz_clock(clk)
        print("   stamps (cycles since start, CTA 0):", list(clk)[:12], "newton it0:", list(clk)[16:21])
