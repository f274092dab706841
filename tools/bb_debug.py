"""Debug the batch-blocked pair kernel: B = identity, so C[i,j,p] = A[i,j,p]."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1606_05696_b200 import _lib
from paper_1606_05696_b200.kernels import core_call
M, N, K, P = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 256, 32, 4
# A[b, k, m] : apt=1, acs=P, ars=P*K
A = torch.arange(P * K * M, dtype=torch.float32, device="cuda") + 1
B = torch.zeros(K * N, dtype=torch.float32, device="cuda")
for l in range(K):
    B[l + l * K] = 1.0
C = torch.full((M * N * P,), -7.0, dtype=torch.float32, device="cuda")
core_call(M, N, K, 1.0, A, 0, P * K, P, 1, B, 0, 1, K, 0, 0.0, C, 0, 1, M, M * N, P)
torch.cuda.synchronize()
print("kernel", _lib.last_kernel())
a = A.cpu().numpy().reshape(M, K, P)      # a[m, k, b] = A[b + P*k + P*K*m]
c = C.cpu().numpy().reshape(P, N, M)      # c[p, j, i]
want = np.zeros((P, N, M), np.float32)
for p in range(P):
    for j in range(K):
        want[p, j, :] = a[:, j, p]
bad = np.argwhere(c != want)
print("bad", len(bad), "of", c.size)
inv = {float(v): idx for idx, v in np.ndenumerate(a)}
for p, j, i in bad[:40]:
    g = float(c[p, j, i])
    print(f"C[i={i},j={j},b={p}] got {g} want {want[p,j,i]} -> A(m,k,b)={inv.get(g)}")
