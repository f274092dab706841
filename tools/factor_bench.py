"""Time the HOOI factor-update pieces with CUDA events (SBT_GA_DEBUG picks how
far sbt_hooi_factor runs: 1 = W, 2 = W + Z, 0 = all) on the 512^3 rank-32
partial cores, plus the acc64 core product and the status kernel."""
import ctypes, os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1606_05696_b200 import _lib, tucker as tk
from paper_1606_05696_b200.layout import DenseTensor
rng = np.random.default_rng(0)
P = ctypes.c_void_p
tag = os.environ.get("SBT_GA_DEBUG", "0")


def ev(fn, reps=20):
    """Device time per call: `reps` calls captured in one CUDA graph, replayed."""
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


for dims, mode in (((512, 32, 32), 0), ((32, 512, 32), 1), ((32, 32, 512), 2)):
    t = DenseTensor.from_array(rng.standard_normal(dims), dtype="float32")
    # warm start = the leading subspace (the HOOI regime: Newton, no Jacobi)
    x = t.view().double()
    ym = torch.movedim(x, mode, 0).reshape(512, -1)
    warm = torch.linalg.eigh(ym @ ym.t())[1][:, -32:].flip(1).contiguous()
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    us = ev(lambda: tk._factor_device(t, mode, 32, warm, st, 0))
    line = f"mode {mode} debug={tag}: factor {us:.1f} us"
    if mode == 2 and tag == "0":
        line += f"; acc64 core {ev(lambda: tk._mode_product_acc64(t, warm, 2)):.1f} us"
        out = torch.empty(4, dtype=torch.float64, device="cuda")
        line += f"; status {ev(lambda: tk._hooi_status(t, st, out)):.1f} us"
    print(line, flush=True)
