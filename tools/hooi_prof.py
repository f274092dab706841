"""Attribute HOOI iteration time (fp32 512^3 r32) to its functions (synced wrappers)."""
import sys, time, collections
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
T = collections.defaultdict(float); C = collections.Counter()
def wrap(name):
    f = getattr(tk, name)
    def w(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); out = f(*a, **k); torch.cuda.synchronize()
        T[name] += time.perf_counter() - t0; C[name] += 1
        return out
    setattr(tk, name, w)
sbt.hooi(t, (r, r, r), max_iters=2, tol=-1.0)
for name in ("_mode_product", "gram_of_unfolding", "top_eigh", "_sign_fix", "_norm", "_orthonormal", "_gemm64"):
    wrap(name)
for iters in (1, 4):
    T.clear(); C.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sbt.hooi(t, (r, r, r), max_iters=iters, tol=-1.0); torch.cuda.synchronize()
    print(f"iters={iters} total {1e3*(time.perf_counter()-t0):.2f} ms")
    for k in T: print(f"   {k:20s} {C[k]:3d} calls {1e3*T[k]:8.2f} ms")
