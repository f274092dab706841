"""Per-phase timing of one HOOI iteration (fast path), bench configs[3] data."""
import sys, time
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
model = sbt.hooi(t, (r, r, r), max_iters=2, tol=-1.0)
f = list(model.factors)
T = {}
def ph(name, fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
    T[name] = T.get(name, 0) + (time.perf_counter() - t0) * 1e3; return out
for rep in range(3):
    y = ph("chain skip0", lambda: tk._mode_product_chain(t, f, skip=0, transpose=True))
    gm = ph("gram0", lambda: tk.gram_of_unfolding(y, 0))
    tk.SWEEP_LOG.clear()
    v = ph("eig0", lambda: tk.top_eigh(gm, r, q0=f[0]))
    f[0] = tk._sign_fix(v[1].contiguous())
    x0 = ph("x0", lambda: tk._mode_product(t, f[0], 0, True))
    y = ph("y(x0 x2)", lambda: tk._mode_product(x0, f[2], 2, True))
    gm = ph("gram1", lambda: tk.gram_of_unfolding(y, 1))
    v = ph("eig1", lambda: tk.top_eigh(gm, r, q0=f[1])); f[1] = tk._sign_fix(v[1].contiguous())
    y2 = ph("y2(x0 x1)", lambda: tk._mode_product(x0, f[1], 1, True))
    gm = ph("gram2", lambda: tk.gram_of_unfolding(y2, 2))
    v = ph("eig2", lambda: tk.top_eigh(gm, r, q0=f[2])); f[2] = tk._sign_fix(v[1].contiguous())
    c = ph("core", lambda: tk._mode_product(y2, f[2], 2, True))
    ph("norm", lambda: tk._norm(c))
for k, v in T.items():
    print(f"{k:14s} {v/3:8.3f} ms")
print("total", sum(T.values()) / 3)
print("sweeps", [(c, f"{d:.1e}") for a, b, c, d in tk.SWEEP_LOG])
for m in (1, 3, 5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sbt.hooi(t, (r, r, r), max_iters=m, tol=-1.0); torch.cuda.synchronize()
    print("hooi", m, (time.perf_counter() - t0) * 1e3)
