import sys, time
sys.path.insert(0, ".")
import torch
from paper_1606_05696_b200 import kernels, _lib
from paper_1606_05696_b200.kernels import Op
lib = _lib.load()
for dt in (torch.float64, torch.float32):
    a = torch.rand(512 * 48, device="cuda", dtype=dt); b = torch.rand(512 * 48, device="cuda", dtype=dt); c = torch.empty(48 * 48, device="cuda", dtype=dt)
    f = lambda: kernels.gemm(Op.Transpose, Op.Normal, 48, 48, 512, 1.0, a, 512, b, 512, 0.0, c, 48)
    for _ in range(10): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(1000): f()
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(dt, "kernels.gemm host per call", (t1 - t0) * 1e3, "us; incl. drain", (t2 - t0) * 1e3, "us", _lib.last_kernel())
    fn = lib.sbt_gemm_core_f64 if dt == torch.float64 else lib.sbt_gemm_core_f32
    s = torch.cuda.current_stream().cuda_stream
    pa, pb, pc = a.data_ptr(), b.data_ptr(), c.data_ptr()
    g = lambda: fn(48, 48, 512, 1.0, pa, 0, 512, 1, pb, 0, 1, 512, 0.0, pc, 0, 1, 48, s)
    for _ in range(10): g()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(1000): g()
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(dt, "raw ctypes per call", (t1 - t0) * 1e3, "us; incl. drain", (t2 - t0) * 1e3, "us")
