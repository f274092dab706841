"""Jacobi sweeps / residuals / phase cycles of the device Ritz steps inside
the bench's HOOI (configs[3])."""
import sys
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
for dt in (torch.float32, torch.float64):
    t = DenseTensor(Layout.packed((n, n, n)), x.permute(2, 1, 0).contiguous().reshape(-1).to(dt))
    tk.RITZ_LOG = []
    sbt.hooi(t, (r, r, r), max_iters=4, tol=-1.0)
    torch.cuda.synchronize()
    for i, rel in enumerate(tk.RITZ_LOG):
        v = rel.tolist()
        print(dt, i, f"rel {v[0]:.2e} newton {v[5]:.0f} sweeps {v[1]:.0f} cycles {v[2]:.0f} {v[3]:.0f} {v[4]:.0f}")
