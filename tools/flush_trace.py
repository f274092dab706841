"""Timeline of the CTA-pair kernel on a HOOI T-product (512^3 x_1 U^T, rank
32): run with SBT_LIB = a -DSBT_TRACE build; compare SBT_TC_FLUSH=0/1."""
import ctypes, sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1606_05696_b200 import _lib, tucker as tk
from paper_1606_05696_b200.layout import DenseTensor, Layout
lib = _lib.load()
n, r = 512, 32
t = DenseTensor(Layout.packed((n, n, n)), torch.randn(n ** 3, device="cuda"))
u = torch.linalg.qr(torch.randn(n, r, dtype=torch.float64, device="cuda"))[0]
for _ in range(3):
    tk._mode_product(t, u, 1, True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); tk._mode_product(t, u, 1, True); e1.record(); torch.cuda.synchronize()
print(f"product: {e0.elapsed_time(e1) * 1e3:.1f} us ({_lib.last_kernel()})")
tr = np.zeros((8, 4096), dtype=np.int64)
fl = np.zeros((2, 4096), dtype=np.int64)
ep = np.zeros((2, 64, 4), dtype=np.int64)
mm = np.zeros((64, 2), dtype=np.int64)
for which, arr in ((0, tr), (1, fl), (2, ep), (3, mm)):
    lib.sbt_trace_dump(which, arr.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
t0 = tr[3][0] if tr[3][0] else tr[0][0]
names = ["tma_free", "landed", "conv_done", "mma_full", "r1_tma_free", "r1_landed", "r1_conv_done", "issue_done"]
for row in (0, 1, 2, 3, 7):
    x = tr[row][tr[row] > 0]
    if len(x) > 40:
        d = np.diff(x[16:len(x) - 8])
        print(f"{names[row]:12s} n={len(x):5d} median interval {np.median(d):7.0f} cyc  mean {d.mean():7.0f}")
for rk in (0, 1):
    x = fl[rk][fl[rk] > 0]
    if len(x) > 10:
        d = np.diff(x[4:])
        print(f"flush rank{rk}  n={len(x)} median group interval {np.median(d):.0f} mean {d.mean():.0f}")
for rk in (0, 1):
    for k in range(4):
        if ep[rk][k][0]:
            print(f"rank{rk} tile{k}: epi begin {ep[rk][k][0] - t0} dur {ep[rk][k][1] - ep[rk][k][0]} "
                  f"tmem_ld {ep[rk][k][2]} rest {ep[rk][k][3]}")
print("mma tiles (acquired, last commit):", [(int(a - t0), int(b - t0)) for a, b in mm[:6] if a])
# K-block timeline excerpt around the 3rd tile
kb = 16 * 3
for row in (0, 1, 2, 3, 7):
    print(f"{names[row]:12s}", " ".join(str(int(v - t0)) for v in tr[row][kb:kb + 12]))
print("flush r0   ", " ".join(str(int(v - t0)) for v in fl[0][8 * 3 // 1: 8 * 3 + 10]))
