import sys, time
sys.path.insert(0, ".")
import torch
import paper_1606_05696_b200 as sbt
from paper_1606_05696_b200 import tucker as tk
from paper_1606_05696_b200.layout import DenseTensor, Layout
n, r = 512, 32
t = DenseTensor(Layout.packed((n, n, n)), torch.randn(n ** 3, device="cuda"))
def timed(name, fn, reps=3):
    out = fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): out = fn()
    torch.cuda.synchronize(); print(f"{name:36s} {(time.perf_counter()-t0)/reps*1e3:8.2f} ms", flush=True); return out
for m in range(3):
    g = timed(f"gram mode {m} of T (fp32->fp64)", lambda: tk.gram_of_unfolding(t, m))
timed("top_eigh cold (noise Gram)", lambda: tk.top_eigh(g, r))
timed("norm T", lambda: tk._norm(t))
timed("hooi 1 iter", lambda: sbt.hooi(t, (r, r, r), max_iters=1, tol=-1.0), reps=1)
timed("hooi 3 iter", lambda: sbt.hooi(t, (r, r, r), max_iters=3, tol=-1.0), reps=1)
