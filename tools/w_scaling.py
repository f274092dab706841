"""Device time of the w_kernel (sbt_mode_product_acc64_f32, mode 0) vs the
number of unfolding columns, next to a trivial torch kernel in the same kind
of graph: separates fixed per-launch cost from per-CTA work."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1606_05696_b200 import tucker as tk
from paper_1606_05696_b200.layout import DenseTensor


def ev(fn, reps=20):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.capture_begin()
        for _ in range(reps):
            fn()
        g.capture_end()
    torch.cuda.current_stream().wait_stream(s)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * reps) * 1e3


x = torch.zeros(16, device="cuda")
print(f"torch add_ on 16 floats: {ev(lambda: x.add_(1.0)):.2f} us")
u = torch.linalg.qr(torch.randn(512, 32, dtype=torch.float64, device="cuda"))[0]
for cols in (32, 128, 512, 1024, 4096):
    t = DenseTensor.from_array(np.random.default_rng(0).standard_normal((512, cols)), dtype="float32")
    print(f"w_kernel n=512 p=32 cols={cols}: {ev(lambda: tk._mode_product_acc64(t, u, 0)):.2f} us", flush=True)
for n in (64, 128, 256):
    t = DenseTensor.from_array(np.random.default_rng(0).standard_normal((n, 1024)), dtype="float32")
    un = torch.linalg.qr(torch.randn(n, 32, dtype=torch.float64, device="cuda"))[0]
    print(f"w_kernel n={n} p=32 cols=1024: {ev(lambda: tk._mode_product_acc64(t, un, 0)):.2f} us", flush=True)

from paper_1606_05696_b200 import _lib
import ctypes
lib = _lib.load()
if hasattr(lib, "sbt_ga_clock"):
    t = DenseTensor.from_array(np.random.default_rng(0).standard_normal((512, 1024)), dtype="float32")
    tk._mode_product_acc64(t, u, 0); torch.cuda.synchronize()
    clk = (ctypes.c_longlong * 16)()
    lib.sbt_ga_clock(clk)
    print("w_kernel stamps (cycles): setup, issued, landed, synced, dmma, end:", list(clk)[:6])
    y = DenseTensor.from_array(np.random.default_rng(0).standard_normal((512, 32, 32)), dtype="float32")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    tk._factor_device(y, 0, 32, u, st, 0); torch.cuda.synchronize()
    lib.sbt_ga_clock(clk)
    print("z_kernel stamps (cycles): colb, loads issued, landed, dmma, cluster sync, reduced, end:",
          list(clk)[8:15])
