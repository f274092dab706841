"""Where does a HOOI iteration's time go? (configs[3], 512^3 rank 32 fp32)"""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1606_05696_b200 as sbt
from paper_1606_05696_b200 import tucker as tk
from paper_1606_05696_b200.layout import DenseTensor, Layout
sys.argv += ["512"]
n, r = int(sys.argv[1]), 32
g = torch.Generator(device="cuda").manual_seed(0)
core = torch.randn(r, r, r, device="cuda", generator=g, dtype=torch.float64)
us = [torch.linalg.qr(torch.randn(n, r, device="cuda", generator=g, dtype=torch.float64))[0] for _ in range(3)]
x = torch.einsum("ia,abc->ibc", us[0], core); x = torch.einsum("jb,ibc->ijc", us[1], x); x = torch.einsum("kc,ijc->ijk", us[2], x)
x = x + 1e-3 * torch.randn(n, n, n, device="cuda", generator=g, dtype=torch.float64)
t = DenseTensor(Layout.packed((n, n, n)), x.permute(2, 1, 0).contiguous().reshape(-1).to(torch.float32))
del x
model = sbt.hooi(t, (r, r, r), max_iters=1, tol=-1.0)
f = model.factors

def timed(name, fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    print(f"{name:40s} {(time.perf_counter()-t0)/reps*1e3:9.3f} ms", flush=True)
    return out

y = timed("chain skip0 (2 products)", lambda: tk._mode_product_chain(t, f, skip=0, transpose=True))
gm = timed("gram mode0 of y (512x512, K=1024)", lambda: tk.gram_of_unfolding(y, 0))
timed("gram mode1 of y (unfold copy)", lambda: tk.gram_of_unfolding(y, 1))
timed("torch.linalg.eigh 512 fp64", lambda: torch.linalg.eigh(gm))
timed("jacobi_eigh (incl. checks)", lambda: tk.jacobi_eigh(gm))
timed("_factor_from_tensor(y,0)", lambda: tk._factor_from_tensor(y, 0, r))
timed("x0 = T x0 U0^T", lambda: tk._mode_product(t, f[0], 0, True))
timed("norm", lambda: tk._norm(t))
timed("hooi 1 iter", lambda: sbt.hooi(t, (r, r, r), max_iters=1, tol=-1.0), reps=2)
timed("hooi 3 iters", lambda: sbt.hooi(t, (r, r, r), max_iters=3, tol=-1.0), reps=2)
from paper_1606_05696_b200 import _lib
print("tf32 UMMA peak TFLOP/s:", [round(_lib.probe_tf32_peak(), 1) for _ in range(3)])
print("dmma peak TFLOP/s:", round(_lib.probe_fp64_peak("dmma"), 2))
tk.SWEEP_LOG.clear()
sbt.hooi(t, (r, r, r), max_iters=3, tol=-1.0)
print("sweep log:", [(a, c, f"{d:.1e}") for a, b, c, d in tk.SWEEP_LOG])
