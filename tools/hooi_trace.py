"""Kernel-level trace of HOOI iterations (torch.profiler, CUPTI): which
kernels run, how long, and how much of the wall time the GPU is idle."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1606_05696_b200 as sbt
from paper_1606_05696_b200.layout import DenseTensor, Layout
n, r = 512, 32
g = torch.Generator(device="cuda").manual_seed(0)
core = torch.randn(r, r, r, device="cuda", generator=g, dtype=torch.float64)
us = [torch.linalg.qr(torch.randn(n, r, device="cuda", generator=g, dtype=torch.float64))[0] for _ in range(3)]
x = torch.einsum("ia,abc->ibc", us[0], core); x = torch.einsum("jb,ibc->ijc", us[1], x); x = torch.einsum("kc,ijc->ijk", us[2], x)
x = x + 1e-3 * torch.randn(n, n, n, device="cuda", generator=g, dtype=torch.float64)
t = DenseTensor(Layout.packed((n, n, n)), x.permute(2, 1, 0).contiguous().reshape(-1).to(torch.float32))
del x
sbt.hooi(t, (r, r, r), max_iters=5, tol=-1.0)   # captures the iteration graph (cached)
from torch.profiler import profile, ProfilerActivity
from collections import defaultdict


def run(iters):
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        sbt.hooi(t, (r, r, r), max_iters=iters, tol=-1.0)
        torch.cuda.synchronize()
    tot = defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot[e.name][0] += 1
            tot[e.name][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    return tot


a, b = run(1), run(5)
rows = []
for k in b:
    c = b[k][0] - a.get(k, [0, 0])[0]
    us = b[k][1] - a.get(k, [0, 0])[1]
    rows.append((us / 4, c / 4, k))
rows.sort(reverse=True)
print("per iteration (5-iter run minus 1-iter run, / 4):")
for us, c, k in rows[:30]:
    print(f"{us:9.1f} us {c:6.1f}x  {k[:110]}")
print("GPU busy per iter", sum(x[0] for x in rows), "us")
for m in (1, 5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sbt.hooi(t, (r, r, r), max_iters=m, tol=-1.0); torch.cuda.synchronize()
    print("wall hooi", m, (time.perf_counter() - t0) * 1e3)

# per-launch durations of one iteration (the last 5-iteration run's final iteration)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sbt.hooi(t, (r, r, r), max_iters=3, tol=-1.0)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
tail = evs[-40:]
print("last launches (us):")
for e in tail:
    d = e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    print(f"  {d:8.1f}  {e.name[:90]}")
