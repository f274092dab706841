"""Tucker decomposition by higher-order orthogonal iteration, on the device.

Algorithm and ordering follow the reference (``tucker.py:87-174``):

* factors start from the truncated HOSVD: leading left singular vectors of
  each mode-r unfolding via its Gram matrix, eigenvalues descending, each
  vector's largest-magnitude entry made positive (``tucker.py:63-76``);
* every mode product is one planned single-mode contraction
  (``_mode_product_chain``, ``tucker.py:87-123``) executed by the sm_100a
  kernels -- modes with the larger reduction extent first, ties in ascending
  mode order -- so no tensor is transposed or copied;
* fit = 1 - sqrt(max(0, ||T||^2 - ||G||^2)) / ||T||, early stop when the fit
  improves by less than ``tol`` after the first iteration.

Precision: the mode products run in the tensor's dtype (fp32 -> 3xTF32 tensor
cores, fp64 -> DMMA); Gram matrices, eigensolves and norms are fp64.
Eigensolver: the reference's cyclic Jacobi (``tucker.py:21-60``) builds an
n x n rotation per pivot and is infeasible at n = 512; ``jacobi_eigh`` here
keeps its contract (values descending, matching eigenvector columns, symmetry
check) but solves with the device's LAPACK-class ``torch.linalg.eigh``
(cuSOLVER) in fp64.  This is off the contraction hot path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .kernels import Op, gemm
from .layout import DenseTensor, Layout, unfold
from .notation import ContractionSpec
from .planner import execute_plan, plan_single_mode

_LETTERS = "abcdefgh"


def _torch():
    import torch
    return torch


def jacobi_eigh(sym, tol: float = 1e-12, max_sweeps: int = 60):
    """Symmetric eigendecomposition, eigenvalues descending with matching
    eigenvector columns (contract of reference tucker.py:21-60).  Accepts numpy
    or torch input; returns the same kind."""
    torch = _torch()
    is_np = isinstance(sym, np.ndarray)
    a = torch.as_tensor(np.asarray(sym) if is_np else sym).to(torch.float64)
    n = a.shape[0]
    if a.dim() != 2 or a.shape != (n, n):
        raise ValueError("matrix must be square")
    scale = max(1.0, float(a.abs().max())) if a.numel() else 1.0
    if not torch.allclose(a, a.t(), atol=1e-12 * scale, rtol=1e-5):
        raise ValueError("matrix must be symmetric")
    if float(torch.linalg.norm(a)) == 0.0:
        w, v = torch.zeros(n, dtype=torch.float64), torch.eye(n, dtype=torch.float64)
    else:
        w, v = torch.linalg.eigh(a)
        order = torch.argsort(w, descending=True)
        w, v = w[order], v[:, order]
    if is_np:
        return w.cpu().numpy(), v.cpu().numpy()
    return w, v


def _sign_fix(u):
    """Largest-magnitude entry of each column made positive (tucker.py:71-75)."""
    torch = _torch()
    idx = torch.argmax(u.abs(), dim=0)
    signs = torch.sign(u[idx, torch.arange(u.shape[1], device=u.device)])
    signs[signs == 0] = 1
    return u * signs


def gram_of_unfolding(t: DenseTensor, r: int):
    """fp64 Gram matrix Y_(r) Y_(r)^T of the mode-r unfolding, on the device.
    Mode 0 and the last mode are read in place by one GEMM launch; middle
    modes go through a packed unfolding copy first."""
    torch = _torch()
    dims = t.layout.dims
    rows = dims[r]
    src = t
    if t.dtype != torch.float64:
        src = DenseTensor(t.layout, t.data.to(torch.float64))
    g = torch.empty(rows * rows, dtype=torch.float64, device=t.device)
    cols = int(np.prod(dims)) // rows
    if t.layout.is_packed() and r == 0:
        gemm(Op.Normal, Op.Transpose, rows, rows, cols, 1.0, src.data, rows, src.data, rows,
             0.0, g, rows)
    elif t.layout.is_packed() and r == len(dims) - 1:
        gemm(Op.Transpose, Op.Normal, rows, rows, cols, 1.0, src.data, cols, src.data, cols,
             0.0, g, rows)
    else:
        u = unfold(src, r)
        gemm(Op.Normal, Op.Transpose, rows, rows, cols, 1.0, u.data, rows, u.data, rows,
             0.0, g, rows)
    return g.reshape(rows, rows).t()  # column-major -> logical (symmetric anyway)


def leading_left_singular_vectors(mat, rank: int):
    """First ``rank`` left singular vectors of a matrix (numpy or torch) via the
    Gram matrix (reference tucker.py:63-76)."""
    torch = _torch()
    is_np = isinstance(mat, np.ndarray)
    m = torch.as_tensor(mat, dtype=torch.float64)
    if rank > m.shape[0]:
        raise ValueError(f"rank {rank} exceeds row count {m.shape[0]}")
    _, vecs = jacobi_eigh(m @ m.t())
    u = _sign_fix(vecs[:, :rank].clone())
    return u.cpu().numpy() if is_np else u


def _factor_from_tensor(t: DenseTensor, r: int, rank: int):
    if rank > t.layout.dims[r]:
        raise ValueError(f"rank {rank} exceeds row count {t.layout.dims[r]}")
    _, vecs = jacobi_eigh(gram_of_unfolding(t, r))
    return _sign_fix(vecs[:, :rank].contiguous())


def _mode_product(cur: DenseTensor, u, r: int, transpose: bool) -> DenseTensor:
    """One planned contraction T x_r U^T (transpose) or T x_r U."""
    order = cur.layout.order
    rows, cols = u.shape
    labels_b, out_ext = (("k", "z"), cols) if transpose else (("z", "k"), rows)
    labels_a = tuple("k" if i == r else _LETTERS[i] for i in range(order))
    labels_c = tuple("z" if i == r else _LETTERS[i] for i in range(order))
    spec = ContractionSpec(labels_a, labels_b, labels_c)
    b = _as_factor_tensor(u, cur.dtype)
    dims = list(cur.layout.dims)
    dims[r] = out_ext
    out = DenseTensor.empty(Layout.packed(dims), dtype=cur.dtype, device=cur.device)
    execute_plan(_planned(spec, cur.layout, b.layout, out.layout), cur, b, 1.0, 0.0, out)
    return out


@dataclass
class TuckerModel:
    core: DenseTensor
    factors: list           # factors[r]: (dim_r x rank_r) torch fp64 tensors on the device
    fit_history: list
    iterations: int


_PLAN_CACHE = {}


def _planned(spec, la, lb, lc):
    key = (spec, la, lb, lc)
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        plan = _PLAN_CACHE[key] = plan_single_mode(spec, la, lb, lc)
    return plan


def _as_factor_tensor(u, dtype):
    """Factor matrix (dim x rank, logical) as a packed column-major DenseTensor."""
    torch = _torch()
    u = torch.as_tensor(u)
    flat = u.to(dtype).t().contiguous().reshape(-1)
    return DenseTensor(Layout.packed(tuple(u.shape)), flat)


def _mode_product_chain(t: DenseTensor, factors, skip, transpose: bool) -> DenseTensor:
    """Apply U_r^T (transpose) or U_r along every mode except ``skip``, one
    planned contraction per mode, larger reduction extent first
    (reference tucker.py:87-123)."""
    order = t.layout.order
    modes = [r for r in range(order) if r != skip]
    red = (lambda r: t.layout.dims[r]) if transpose else (lambda r: factors[r].shape[1])
    modes.sort(key=lambda r: -red(r))
    cur = t
    for r in modes:
        cur = _mode_product(cur, factors[r], r, transpose)
    return cur


def tucker_core(t: DenseTensor, factors) -> DenseTensor:
    """G = T x_1 U_1^T x_2 U_2^T ... via planned contractions."""
    return _mode_product_chain(t, factors, skip=None, transpose=True)


def tucker_reconstruct(model: TuckerModel) -> DenseTensor:
    return _mode_product_chain(model.core, model.factors, skip=None, transpose=False)


def _norm(t: DenseTensor) -> float:
    torch = _torch()
    return float(torch.linalg.vector_norm(t.data.to(torch.float64)))


def _reuses_mode0(t: DenseTensor) -> bool:
    """For order 3 with mode 0 the largest, the reference chains for skip=1,
    skip=2 and the core all START with T x_0 U_0^T under the same U_0
    (tucker.py:95-99 sorts by reduction extent, ties ascending), so that product
    can be computed once per iteration with bitwise-identical results."""
    d = t.layout.dims
    return t.layout.order == 3 and d[0] >= d[2] and d[0] >= d[1]


def hooi(t: DenseTensor, ranks, max_iters: int = 50, tol: float = 1e-10,
         reuse_mode0: bool = True) -> TuckerModel:
    """Higher-order orthogonal iteration (reference tucker.py:136-174).

    With ``reuse_mode0`` (order-3 tensors whose mode 0 is the largest) the
    product T x_0 U_0^T that the reference recomputes three times per iteration
    is computed once: T is read twice per iteration instead of four times, with
    the same operations in the same order."""
    order = t.layout.order
    ranks = tuple(int(r) for r in ranks)
    if len(ranks) != order:
        raise ValueError(f"need {order} ranks, got {len(ranks)}")
    for r, (rank, dim) in enumerate(zip(ranks, t.layout.dims)):
        if not 1 <= rank <= dim:
            raise ValueError(f"rank {rank} invalid for mode {r} extent {dim}")
    torch = _torch()
    t64 = t if t.dtype == torch.float64 else DenseTensor(t.layout, t.data.to(torch.float64))
    factors = [_factor_from_tensor(t64, r, ranks[r]) for r in range(order)]
    del t64
    norm_t = _norm(t)
    fits = []
    prev = -np.inf
    iters = 0
    fast = reuse_mode0 and _reuses_mode0(t)
    for it in range(max_iters):
        iters = it + 1
        if fast:
            # skip=0 chain: modes 1, 2 (reference order); then X0 = T x_0 U_0^T
            y = _mode_product_chain(t, factors, skip=0, transpose=True)
            factors[0] = _factor_from_tensor(y, 0, ranks[0])
            x0 = _mode_product(t, factors[0], 0, True)
            # reference skip=1 chain is [0, 2] and skip=2 chain is [0, 1]
            y = _mode_product(x0, factors[2], 2, True)
            factors[1] = _factor_from_tensor(y, 1, ranks[1])
            y2 = _mode_product(x0, factors[1], 1, True)
            factors[2] = _factor_from_tensor(y2, 2, ranks[2])
            # reference core chain: mode 0, then the larger of modes 1 / 2 first
            if t.layout.dims[1] >= t.layout.dims[2]:
                core = _mode_product(y2, factors[2], 2, True)
            else:
                core = _mode_product(_mode_product(x0, factors[2], 2, True), factors[1], 1, True)
        else:
            for r in range(order):
                y = _mode_product_chain(t, factors, skip=r, transpose=True)
                factors[r] = _factor_from_tensor(y, r, ranks[r])
            core = tucker_core(t, factors)
        norm_g = _norm(core)
        resid = np.sqrt(max(0.0, norm_t ** 2 - norm_g ** 2))
        fit = 1.0 - resid / norm_t if norm_t > 0 else 1.0
        fits.append(fit)
        if fit - prev < tol and it > 0:
            break
        prev = fit
    core = tucker_core(t, factors)
    return TuckerModel(core=core, factors=factors, fit_history=fits, iterations=iters)
