import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1606_05696_b200 as sbt
from paper_1606_05696_b200 import tucker as tk
from paper_1606_05696_b200.layout import DenseTensor
from oracle import tucker as otucker
rng = np.random.default_rng(10)
dims, ranks = (160, 144, 136), (8, 8, 6)
core = rng.standard_normal(ranks)
us = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
full = np.einsum("abc,ia,jb,kc->ijk", core, *us) + 1e-3 * rng.standard_normal(dims)
t = DenseTensor.from_array(full, dtype="float32")
ref = otucker.hooi(t.to_array().astype(np.float64), ranks, max_iters=3, tol=-1.0)
for minn in (128, 10**9):
    tk._SUBSPACE_MIN_N = minn
    model = sbt.hooi(t, ranks, max_iters=3, tol=-1.0)
    print("min_n", minn, "fit", model.fit_history, "ref", ref["fit_history"])
tk._SUBSPACE_MIN_N = 128
# timing of the eigensolver at 512
x = torch.randn(512, 32, device="cuda", dtype=torch.float64) @ torch.randn(32, 2048, device="cuda", dtype=torch.float64)
x += 1e-3 * torch.randn(512, 2048, device="cuda", dtype=torch.float64)
g = x @ x.t()
for warm in (None, "warm"):
    q0 = None if warm is None else tk.top_eigh(g, 32)[1]
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5):
        w, v, its = tk.top_eigh(g, 32, q0=q0)
    torch.cuda.synchronize(); print("top_eigh", warm, its, "sweeps", (time.perf_counter() - t0) / 5 * 1e3, "ms")
z = torch.randn(48, 512, device="cuda", dtype=torch.float64)
for f, name in ((lambda: tk._orthonormal(z), "qr"), (lambda: g.cpu(), "d2h 2MB"), (lambda: z[:2].cpu(), "d2h small")):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(10): f()
    torch.cuda.synchronize(); print(name, (time.perf_counter() - t0) / 10 * 1e3, "ms")
