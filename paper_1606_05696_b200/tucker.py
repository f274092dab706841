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
(cuSOLVER) in fp64; HOOI's warm factor updates instead finish their subspace
sweeps on the device (``_factor_device``, k_ritz.cuh), one host round trip per
iteration, replayed as a CUDA graph (``_IterationGraph``).
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


# Leading-eigenvector solver for the HOOI Grams.  Only the top ``rank``
# eigenpairs of an n x n PSD Gram are needed (tucker.py:69-70 keeps the first
# ``rank`` columns), so for n >= _SUBSPACE_MIN_N the factor comes from block
# subspace iteration with Rayleigh-Ritz, warm-started from the previous HOOI
# factor: every n-sized product is an fp64 GEMM on the sm_100a kernels, the
# (rank+oversample)^2 projected problem is solved on the host, and the loop
# stops when every kept Ritz pair has ||G u - w u|| <= tol * w_max -- the
# accuracy of a full eigh.  If it has not converged after _SUBSPACE_MAX_IT
# sweeps (small eigengap), the full eigendecomposition is used instead.
_SUBSPACE_MIN_N = 128
_SUBSPACE_MAX_IT = 40
_SUBSPACE_TOL = 1e-12
# fp32 tensors: the mode products feeding the Gram are fp32 (3xTF32: relative
# error ~2e-6 at K = 512), and from one HOOI iteration to the next that noise
# alone moves the leading subspace by ~5e-8 (measured residual floor of a
# warm sweep at 512^3, rank 32), so Ritz pairs with residual <= 1e-6 * w_max
# are at data precision; a tighter test would only flag the noise
_SUBSPACE_TOL_F32 = 1e-6
SWEEP_LOG = []  # (n, rank, sweep, max relative residual): diagnostics only


def _gemm64(opa, opb, m, n, k, a, lda, b, ldb, c, ldc, alpha=1.0, beta=0.0):
    """fp64 GEMM on the device through the library (column-major flat views)."""
    gemm(opa, opb, m, n, k, alpha, a.reshape(-1), lda, b.reshape(-1), ldb, beta,
         c.reshape(-1), ldc)


def _orthonormal(z):
    """Orthonormal basis of the columns of z (n x p, column-major as a (p, n)
    row-major torch tensor): Householder QR (cuSOLVER)."""
    torch = _torch()
    q, _ = torch.linalg.qr(z.t())
    return q.t().contiguous()


def top_eigh(g, rank: int, q0=None, tol: float = _SUBSPACE_TOL,
             max_iter: int = _SUBSPACE_MAX_IT):
    """Top ``rank`` eigenpairs (descending) of the symmetric PSD matrix ``g``
    (torch fp64, n x n, on the device).  Returns (w[rank], V[n, rank]) and the
    number of subspace sweeps (0 = full eigh was used)."""
    torch = _torch()
    n = g.shape[0]
    if n < _SUBSPACE_MIN_N or 4 * rank > n:
        w, v = jacobi_eigh(g)
        return w[:rank], v[:, :rank], 0
    p_full = min(n, rank + max(8, rank // 2))
    gen = torch.Generator(device=g.device).manual_seed(20260824 + n * 131 + rank)
    # bases are stored transposed: qt[p, n] row-major == Q[n, p] column-major
    if q0 is not None:
        # warm start: the previous (orthonormal) factor alone; oversampling
        # columns are added only if one sweep does not converge
        qt = torch.as_tensor(q0, dtype=torch.float64, device=g.device).t().contiguous()
        expand = True
    else:
        qt = _orthonormal(torch.randn(p_full, n, device=g.device, dtype=torch.float64,
                                      generator=gen))
        expand = False
    gm = g.contiguous()  # symmetric: row-major == column-major
    # residual norms from the projected Gram: with Q orthonormal, u = Q v and
    # G u = Z v, ||G u - w u||^2 = v^T (Z^T Z) v - w^2.  The difference of two
    # O(w^2) numbers resolves r / w down to ~1e-8, so it serves tolerances
    # >= 1e-9 (fp32 tensors) with one device->host copy per sweep; tighter
    # tolerances compute the residual vectors explicitly.
    fast = tol >= 1e-9
    wmax = None
    prev_res = None
    for it in range(1, max_iter + 1):
        p = qt.shape[0]
        qz = torch.empty(2 * p, n, device=g.device, dtype=torch.float64)  # [Q | Z] col-major
        qz[:p] = qt
        zt = qz[p:]
        _gemm64(Op.Normal, Op.Normal, n, p, n, gm, n, qt, n, zt, n)          # Z = G Q
        wqz = torch.empty(p, 2 * p, device=g.device, dtype=torch.float64)
        _gemm64(Op.Transpose, Op.Normal, 2 * p, p, n, qz, n, zt, n, wqz, 2 * p)  # [Q Z]^T Z
        hw = wqz.cpu().numpy()                 # hw[j, i] = ([Q Z]^T Z)[i, j]
        hh, ss = hw[:, :p].T, hw[:, p:].T      # H = Q^T G Q, S = Z^T Z
        w, v = np.linalg.eigh(0.5 * (hh + hh.T))
        order = np.argsort(w)[::-1]
        w, v = w[order], v[:, order]
        wmax = max(float(w[0]), 0.0)
        if wmax == 0.0:
            break
        vt = torch.as_tensor(np.ascontiguousarray(v.T), device=g.device)  # V col-major (ld p)
        ut = torch.empty_like(qt)
        _gemm64(Op.Normal, Op.Normal, n, p, p, qt, n, vt, p, ut, n)        # U = Q V
        wt = torch.as_tensor(w[:rank].copy(), device=g.device)
        if fast:
            vr = v[:, :rank]
            r2 = np.einsum("ij,ik,kj->j", vr, 0.5 * (ss + ss.T), vr) - w[:rank] ** 2
            rmax = float(np.sqrt(max(0.0, r2.max())))
            yt = None
        else:
            yt = torch.empty_like(qt)
            _gemm64(Op.Normal, Op.Normal, n, p, p, zt, n, vt, p, yt, n)    # Y = G U
            res = torch.linalg.vector_norm(yt[:rank] - wt[:, None] * ut[:rank], dim=1)
            rmax = float(res.max())
        SWEEP_LOG.append((n, rank, it, rmax / wmax))
        if rmax <= tol * wmax:
            return (wt, ut[:rank].t().contiguous(), it)
        # give up early when the observed contraction rate cannot reach tol in
        # a few more sweeps (small eigengap): the full solver is cheaper then
        if prev_res is not None and it >= 3:
            rate = rmax / prev_res
            need = np.log(tol * wmax / rmax) / np.log(rate) if 0 < rate < 1 else np.inf
            if need > 6:
                break
        prev_res = rmax
        if yt is None:
            yt = torch.empty_like(qt)
            _gemm64(Op.Normal, Op.Normal, n, p, p, zt, n, vt, p, yt, n)    # Y = G U
        if expand and p < p_full:
            extra = torch.randn(p_full - p, n, device=g.device, dtype=torch.float64,
                                generator=gen)
            qt = _orthonormal(torch.cat([yt, extra]))
            prev_res = None
        else:
            qt = _orthonormal(yt)
        expand = False
    w, v = jacobi_eigh(g)
    return w[:rank], v[:, :rank], 0


def _sign_fix(u):
    """Largest-magnitude entry of each column made positive (tucker.py:71-75)."""
    torch = _torch()
    idx = torch.argmax(u.abs(), dim=0)
    signs = torch.sign(u[idx, torch.arange(u.shape[1], device=u.device)])
    signs[signs == 0] = 1
    return u * signs


def gram_of_unfolding(t: DenseTensor, r: int):
    """fp64 Gram matrix Y_(r) Y_(r)^T of the mode-r unfolding, on the device.

    The Gram does not depend on the order of the unfolding's columns, so any
    buffer with mode r as its unit-stride mode serves.  An fp64 packed tensor
    is read in place for mode 0 and the last mode (one GEMM launch); otherwise
    one fused pass converts to fp64 AND moves mode r to the front (the copy
    the fp32 -> fp64 conversion needs anyway), then one GEMM."""
    torch = _torch()
    dims = t.layout.dims
    rows = dims[r]
    cols = int(np.prod(dims)) // rows
    g = torch.empty(rows * rows, dtype=torch.float64, device=t.device)
    if r in (0, len(dims) - 1):
        if t.dtype == torch.float64 and t.layout.is_packed():
            src = t.data
        else:                                            # one pass: convert / pack
            x = t.view()
            rev = tuple(reversed(range(x.dim())))
            buf = torch.empty(tuple(x.shape[i] for i in rev), dtype=torch.float64,
                              device=t.device)
            buf.copy_(x.permute(rev))
            src = buf.reshape(-1)
        if r == 0:
            gemm(Op.Normal, Op.Transpose, rows, rows, cols, 1.0, src, rows, src, rows,
                 0.0, g, rows)
        else:
            gemm(Op.Transpose, Op.Normal, rows, rows, cols, 1.0, src, cols, src, cols,
                 0.0, g, rows)
    else:
        x = t.view().movedim(r, 0)                       # logical (rows, rest...)
        rev = tuple(reversed(range(x.dim())))
        buf = torch.empty(tuple(x.shape[i] for i in rev), dtype=torch.float64,
                          device=t.device)
        buf.copy_(x.permute(rev))                         # column-major, mode r fastest
        flat = buf.reshape(-1)
        gemm(Op.Normal, Op.Transpose, rows, rows, cols, 1.0, flat, rows, flat, rows,
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


def _factor_from_tensor(t: DenseTensor, r: int, rank: int, warm=None):
    """Leading ``rank`` left singular vectors of the mode-r unfolding: top
    eigenvectors of its fp64 Gram (subspace iteration warm-started from the
    previous factor ``warm`` when given), sign-fixed as tucker.py:71-75."""
    if rank > t.layout.dims[r]:
        raise ValueError(f"rank {rank} exceeds row count {t.layout.dims[r]}")
    torch = _torch()
    tol = _SUBSPACE_TOL if t.dtype == torch.float64 else _SUBSPACE_TOL_F32
    _, vecs, _ = top_eigh(gram_of_unfolding(t, r), rank, q0=warm, tol=tol)
    return _sign_fix(vecs.contiguous())


# Device-finished sweeps (k_ritz.cuh): inside HOOI, a warm-started factor
# update normally converges in ONE subspace sweep (the previous factor spans
# the new leading subspace to ~1e-8).  The sweep's projected eigenproblem,
# Ritz vectors, residual test and sign rule then run in one kernel with no
# host round trip; the convergence flags of all factors are read once per
# iteration together with ||G||, and an iteration with an unconverged factor
# is recomputed on the host-driven path (top_eigh: more sweeps, oversampling,
# full eigh), so results are those of the host path either way.
_RITZ_MAX_P = 64
RITZ_LOG = None  # set to a list to collect each sweep's diagnostics (rel[0..4])


def _ritz_eligible(n: int, rank: int, warm) -> bool:
    return (warm is not None and getattr(warm, "is_cuda", False) and n >= _SUBSPACE_MIN_N
            and 4 * rank <= n and rank <= _RITZ_MAX_P)


_FACTOR_WS = {}


def _factor_ws(dev, dims, r, p):
    """Workspace of sbt_hooi_factor for (dims, mode, p): allocated once per
    device and reused, so a captured iteration allocates nothing."""
    import ctypes
    from . import _lib
    torch = _torch()
    # one workspace per stream (concurrent HOOIs on different streams must not
    # share it), bounded: a long-lived process cycling through shapes keeps the
    # most recent ones
    key = (dev, torch.cuda.current_stream(dev).cuda_stream, tuple(dims), r, p)
    ws = _FACTOR_WS.get(key)
    if ws is None:
        if len(_FACTOR_WS) >= 64:
            _FACTOR_WS.pop(next(iter(_FACTOR_WS)))
        d = (ctypes.c_int64 * len(dims))(*dims)
        nbytes = int(_lib.load().sbt_hooi_factor_ws_bytes(len(dims), d, r, p))
        if nbytes <= 0:
            raise ValueError(f"sbt_hooi_factor_ws_bytes: bad geometry {dims} mode {r} p {p}")
        ws = _FACTOR_WS[key] = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    return ws


def _factor_device(t: DenseTensor, r: int, rank: int, warm, status, slot: int,
                   sweeps: int = 1, out=None):
    """Warm-started subspace sweeps on the mode-r Gram, each finished on the
    device: sweep 1 on the previous factor, further sweeps on the
    orthonormalised G U (one sweep reaches the fp32 tolerance after the first
    HOOI iteration; fp64's 1e-12 takes two).  A sweep is ONE library call
    (``sbt_hooi_factor_*``: G Q = Y (Y^T Q) in fp64 read straight from the
    packed fp32 / fp64 tensor, then the Ritz kernel).  Writes the last sweep's
    convergence flag to status[slot]; never synchronises."""
    import ctypes
    from . import _lib
    torch = _torch()
    fp64 = t.dtype == torch.float64
    tol = _SUBSPACE_TOL if fp64 else _SUBSPACE_TOL_F32
    if not t.layout.is_packed():
        t = DenseTensor(Layout.packed(t.layout.dims), t.view().permute(
            *reversed(range(t.layout.order))).contiguous().reshape(-1))
    dims = tuple(int(d) for d in t.layout.dims)
    n = dims[r]
    dev = t.data.device
    lib = _lib.load()
    ptr = ctypes.c_void_p
    stream = ptr(torch.cuda.current_stream(dev).cuda_stream)
    cdims = (ctypes.c_int64 * len(dims))(*dims)
    entry = lib.sbt_hooi_factor_f64 if fp64 else lib.sbt_hooi_factor_f32
    p = rank
    ws = _factor_ws(dev, dims, r, p)
    qt = torch.as_tensor(warm, device=dev).t()          # (p, n) view: row j = column j
    if qt.stride(1) != 1:
        qt = qt.contiguous()
    for sweep in range(sweeps):
        last = sweep == sweeps - 1
        if last and out is not None:           # caller-owned (rank x n) buffers
            ut, ut32 = out[0], (out[1] if not fp64 else None)
        else:
            ut = torch.empty(rank, n, device=dev, dtype=torch.float64)
            ut32 = (torch.empty(rank, n, device=dev, dtype=torch.float32)
                    if last and not fp64 else None)
        yt = None if last else torch.empty(rank, n, device=dev, dtype=torch.float64)
        w = torch.empty(rank, device=dev, dtype=torch.float64)
        rel = torch.empty(6, device=dev, dtype=torch.float64)
        flag = status[slot:] if last else torch.empty(1, device=dev, dtype=torch.int32)
        _lib.check(entry(
            ptr(t.data.data_ptr()), len(dims), cdims, r, ptr(qt.data_ptr()), qt.stride(0), p,
            rank, float(tol), ptr(ws.data_ptr()), ws.numel(), ptr(ut.data_ptr()),
            ptr(yt.data_ptr() if yt is not None else None),
            ptr(ut32.data_ptr() if ut32 is not None else None), ptr(w.data_ptr()),
            ptr(flag.data_ptr()), ptr(rel.data_ptr()), stream), "sbt_hooi_factor")
        if RITZ_LOG is not None:
            RITZ_LOG.append(rel)              # device tensors: diagnostics only
        if not last:
            qt = _orthonormal(yt)
    u = ut.t()
    if ut32 is not None:
        _attach_f32(u, ut32)       # fp32 copy for the fp32 mode products
    return u


def _hooi_status(core: DenseTensor, status, out):
    """out[0] = ||core||, out[1:] = the factors' flags: one launch
    (``sbt_hooi_status_*``), the iteration's one device->host read."""
    import ctypes
    from . import _lib
    torch = _torch()
    lib = _lib.load()
    ptr = ctypes.c_void_p
    data = core.data if core.layout.is_packed() else core.view().contiguous().reshape(-1)
    entry = lib.sbt_hooi_status_f64 if data.dtype == torch.float64 else lib.sbt_hooi_status_f32
    _lib.check(entry(ptr(data.data_ptr()), data.numel(), ptr(status.data_ptr()), status.numel(),
                     ptr(out.data_ptr()), ptr(torch.cuda.current_stream(data.device).cuda_stream)),
               "sbt_hooi_status")
    return out


# small fp32 products T x_r U^T (at most this many input elements; the HOOI
# core product y2 x_2 U_2^T at 512^3 rank 32 reads 2^19) run with fp64
# accumulation (sbt_mode_product_acc64_f32): the fit compares ||G|| with ||T||
# and amplifies a relative error of ||G|| ~15x (resid / ||T|| ~ 0.064), so the
# core must not carry the tensor core's accumulator truncation (~2e-6 at
# K = 512 on a 128-row tile).  The large products run on the unbiased
# narrow-tile (FLUSH) path of the CTA-pair kernel.
_ACC64_MAX_ELEMS = 1 << 21


def _mode_product_acc64(cur: DenseTensor, u, r: int) -> DenseTensor:
    import ctypes
    from . import _lib
    torch = _torch()
    dims = tuple(int(d) for d in cur.layout.dims)
    rank = int(u.shape[1])
    qt = torch.as_tensor(u, device=cur.data.device, dtype=torch.float64).t()
    if qt.stride(1) != 1:
        qt = qt.contiguous()
    out_dims = list(dims)
    out_dims[r] = rank
    out = DenseTensor.empty(Layout.packed(out_dims), dtype=cur.dtype, device=cur.device)
    lib = _lib.load()
    fn = lib.sbt_mode_product_acc64_f32 if cur.dtype == torch.float32 else \
        lib.sbt_mode_product_acc64_f64
    ptr = ctypes.c_void_p
    _lib.check(fn(ptr(cur.data.data_ptr()), len(dims), (ctypes.c_int64 * len(dims))(*dims), r,
                  ptr(qt.data_ptr()), qt.stride(0), rank, ptr(out.data.data_ptr()),
                  ptr(torch.cuda.current_stream(cur.data.device).cuda_stream)),
               "sbt_mode_product_acc64")
    return out


def _mode_product(cur: DenseTensor, u, r: int, transpose: bool,
                  fast: bool = False) -> DenseTensor:
    """One planned contraction T x_r U^T (transpose) or T x_r U.  ``fast``:
    the product only feeds a factor update (an eigenvector direction, blind to
    the ~K/16-ulp uniform shrink of the tensor core's truncating fp32
    accumulator), so the narrow tiles may skip the unbiased accumulation that
    the products feeding the core -- whose norm the fit compares with ||T|| --
    need (sbt_set_accumulation)."""
    if fast:
        from . import _lib
        with _lib.fast_accumulation():
            return _mode_product(cur, u, r, transpose)
    order = cur.layout.order
    torch = _torch()
    if (transpose and cur.dtype == torch.float32 and cur.layout.is_packed()
            and cur.layout.size <= _ACC64_MAX_ELEMS and u.shape[1] <= 64
            and getattr(u, "is_cuda", False)):
        return _mode_product_acc64(cur, u, r)
    rows, cols = u.shape
    labels_b, out_ext = (("k", "z"), cols) if transpose else (("z", "k"), rows)
    labels_a = tuple("k" if i == r else _LETTERS[i] for i in range(order))
    labels_c = tuple("z" if i == r else _LETTERS[i] for i in range(order))
    spec = ContractionSpec(labels_a, labels_b, labels_c)
    b = _as_factor_tensor(u, cur.dtype, cur.data.device)
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
    stats: dict = None      # path taken per iteration (diagnostics)


_PLAN_CACHE = {}


def _planned(spec, la, lb, lc):
    key = (spec, la, lb, lc)
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        plan = _PLAN_CACHE[key] = plan_single_mode(spec, la, lb, lc)
    return plan


def _attach_f32(u, flat):
    """Keep an fp32 copy (rank x dim, contiguous) of factor ``u`` on the tensor,
    stamped with u's version counter: an in-place change of ``u`` (or of the
    tensor it views) bumps the counter and invalidates the copy."""
    u._sbt_f32 = (u._version, flat)


def _cached_f32(u):
    got = getattr(u, "_sbt_f32", None)
    if got is None or got[0] != u._version:
        return None
    return got[1]


def _as_factor_tensor(u, dtype, device=None):
    """Factor matrix (dim x rank, logical) as a packed column-major DenseTensor
    on ``device`` (numpy factors -- the reference's TuckerModel.factors type --
    are copied there).  The fp32 conversion is made once per factor version
    and kept on the tensor (the device Ritz kernel supplies it directly)."""
    torch = _torch()
    u = torch.as_tensor(u, device=device)
    if dtype == torch.float32:
        flat = _cached_f32(u)
        if flat is None:
            flat = u.to(dtype).t().contiguous()
            if u.is_cuda:
                _attach_f32(u, flat)
        return DenseTensor(Layout.packed(tuple(u.shape)), flat.reshape(-1))
    flat = u.to(dtype).t().contiguous().reshape(-1)
    return DenseTensor(Layout.packed(tuple(u.shape)), flat)


def _mode_product_chain(t: DenseTensor, factors, skip, transpose: bool,
                        fast: bool = False) -> DenseTensor:
    """Apply U_r^T (transpose) or U_r along every mode except ``skip``, one
    planned contraction per mode, larger reduction extent first
    (reference tucker.py:87-123)."""
    order = t.layout.order
    modes = [r for r in range(order) if r != skip]
    red = (lambda r: t.layout.dims[r]) if transpose else (lambda r: factors[r].shape[1])
    modes.sort(key=lambda r: -red(r))
    cur = t
    for r in modes:
        cur = _mode_product(cur, factors[r], r, transpose, fast)
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


def _hooi_sweep(t: DenseTensor, factors, fast: bool, factor_fn) -> DenseTensor:
    """One HOOI iteration (tucker.py:160-167): update every factor in place via
    factor_fn(y, r, warm) and return the core G = T x_1 U_1^T ... x_N U_N^T."""
    order = t.layout.order
    # products that only feed a factor update run with the fast accumulator;
    # those feeding the core (X0, its mode-1 product, the core itself) keep
    # the unbiased one (see _mode_product)
    if fast:
        # skip=0 chain: modes 1, 2 (reference order); then X0 = T x_0 U_0^T
        y = _mode_product_chain(t, factors, skip=0, transpose=True, fast=True)
        factors[0] = factor_fn(y, 0, factors[0])
        x0 = _mode_product(t, factors[0], 0, True)
        # reference skip=1 chain is [0, 2] and skip=2 chain is [0, 1]
        y = _mode_product(x0, factors[2], 2, True, fast=True)
        factors[1] = factor_fn(y, 1, factors[1])
        y2 = _mode_product(x0, factors[1], 1, True)
        factors[2] = factor_fn(y2, 2, factors[2])
        # reference core chain: mode 0, then the larger of modes 1 / 2 first
        if t.layout.dims[1] >= t.layout.dims[2]:
            return _mode_product(y2, factors[2], 2, True)
        return _mode_product(_mode_product(x0, factors[2], 2, True), factors[1], 1, True)
    for r in range(order):
        y = _mode_product_chain(t, factors, skip=r, transpose=True, fast=True)
        factors[r] = factor_fn(y, r, factors[r])
    return tucker_core(t, factors)


class _IterationGraph:
    """The device-finished HOOI iteration captured as a pair of CUDA graphs
    (the iteration is launch-only, so a replay costs no host work).  The
    factors live in two static buffer sets (fp64 rank x n rows, plus their
    fp32 copies for fp32 tensors); graph 0 reads set 0 and its Ritz kernels
    write set 1, graph 1 the reverse, so no factor is ever copied and the
    iteration's starting factors stay intact for a host-path redo.  ``out`` of
    each graph = [||G||, convergence flags...]."""

    # the last captured pair, reused by later hooi() calls on the same tensor
    # buffer and configuration (capture and teardown cost milliseconds; holding
    # the tensor's storage keeps the captured addresses valid)
    _cache = None

    @classmethod
    def get(cls, t, factors, ranks, fast, sweeps):
        key = (t.data.data_ptr(), t.data.dtype, tuple(t.layout.dims), tuple(t.layout.strides),
               tuple(ranks), fast, sweeps, tuple(f.shape for f in factors))
        c = cls._cache
        if c is not None and c[0] == key:
            g = c[1]
            g.load(factors)
            return g
        cls._cache = None
        g = cls.capture(t, factors, ranks, fast, sweeps)
        if g is not None:
            cls._cache = (key, g, t.data)
        return g

    def _views(self, k):
        """Factor views (dim x rank) of buffer set k, with their fp32 copies."""
        vs = []
        for u, u32 in zip(self.sets[k], self.sets32[k]):
            v = u.t()
            if u32 is not None:
                _attach_f32(v, u32)
            vs.append(v)
        return vs

    def load(self, factors):
        """Make ``factors`` the starting point (set ``cur``)."""
        for u, u32, f in zip(self.sets[self.cur], self.sets32[self.cur], factors):
            u.copy_(f.t())
            if u32 is not None:
                u32.copy_(u)

    @property
    def factors(self):
        return self._views(self.cur)

    @classmethod
    def capture(cls, t, factors, ranks, fast, sweeps):
        torch = _torch()
        self = cls()
        order = t.layout.order
        f32 = t.dtype == torch.float32
        self.sets = [[torch.empty(f.shape[1], f.shape[0], device=t.device, dtype=torch.float64)
                      for f in factors] for _ in range(2)]
        self.sets32 = [[torch.empty_like(u, dtype=torch.float32) if f32 else None for u in st]
                       for st in self.sets]
        self.status = [torch.zeros(order, dtype=torch.int32, device=t.device) for _ in range(2)]
        self.out_bufs = [torch.zeros(1 + order, dtype=torch.float64, device=t.device)
                         for _ in range(2)]
        self.out = [None, None]
        self.graphs = [torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()]
        self.cur = 0
        # capture_begin/end on a side stream directly: torch.cuda.graph() would
        # also gc.collect() and empty the caching allocator on every capture
        side = torch.cuda.Stream(device=t.device)
        side.wait_stream(torch.cuda.current_stream(t.device))
        try:
            with torch.cuda.stream(side):
                for k in range(2):
                    self.graphs[k].capture_begin()
                    try:
                        self._record(k, t, ranks, fast, sweeps)
                    finally:
                        self.graphs[k].capture_end()
        except RuntimeError:      # something on the path is not capturable
            torch.cuda.synchronize()
            return None
        torch.cuda.current_stream(t.device).wait_stream(side)
        self.load(factors)
        return self

    def _record(self, k, t, ranks, fast, sweeps):
        st = self.status[k]                # every flag is written by its Ritz kernel
        nxt = 1 - k
        outs = list(zip(self.sets[nxt], self.sets32[nxt]))
        core = _hooi_sweep(t, self._views(k), fast, lambda y, r, warm: _factor_device(
            y, r, ranks[r], warm, st, r, sweeps, out=outs[r]))
        self.out[k] = _hooi_status(core, st, self.out_bufs[k])

    def replay(self):
        """One iteration from set ``cur`` into the other set; returns the
        host copy of [||G||, flags] and advances ``cur`` (``factors`` are then
        the new ones; ``previous`` the starting ones)."""
        k = self.cur
        self.graphs[k].replay()
        vals = self.out[k].cpu().numpy()
        self.cur = 1 - k
        return vals

    @property
    def previous(self):
        return self._views(1 - self.cur)


def clear_graph_cache() -> None:
    """Release the cached HOOI iteration graph (and the tensor it holds)."""
    _IterationGraph._cache = None


def hooi(t: DenseTensor, ranks, max_iters: int = 50, tol: float = 1e-10,
         reuse_mode0: bool = True, device_ritz: bool = True,
         use_graph: bool = True) -> TuckerModel:
    """Higher-order orthogonal iteration (reference tucker.py:136-174).

    With ``reuse_mode0`` (order-3 tensors whose mode 0 is the largest) the
    product T x_0 U_0^T that the reference recomputes three times per iteration
    is computed once: T is read twice per iteration instead of four times, with
    the same operations in the same order.  With ``device_ritz`` the warm
    factor updates finish on the device (see _factor_device) and an iteration
    synchronises with the host once; with ``use_graph`` that iteration is
    captured once as a CUDA graph and replayed (long runs only)."""
    order = t.layout.order
    ranks = tuple(int(r) for r in ranks)
    if len(ranks) != order:
        raise ValueError(f"need {order} ranks, got {len(ranks)}")
    for r, (rank, dim) in enumerate(zip(ranks, t.layout.dims)):
        if not 1 <= rank <= dim:
            raise ValueError(f"rank {rank} invalid for mode {r} extent {dim}")
    torch = _torch()
    factors = [_factor_from_tensor(t, r, ranks[r]) for r in range(order)]
    norm_t = _norm(t)
    fits = []
    prev = -np.inf
    iters = 0
    fast = reuse_mode0 and _reuses_mode0(t)
    host_factor = lambda y, r, warm: _factor_from_tensor(y, r, ranks[r], warm=warm)  # noqa: E731
    graph = None
    stats = {"device_iterations": 0, "host_iterations": 0, "host_redos": 0, "graph": False}
    for it in range(max_iters):
        iters = it + 1
        if device_ritz and all(_ritz_eligible(t.layout.dims[r], ranks[r], factors[r])
                               for r in range(order)):
            sweeps = 2 if (it == 0 or t.dtype == torch.float64) else 1
            if graph is None and use_graph and it >= 1 and max_iters - it >= 3:
                graph = _IterationGraph.get(t, factors, ranks, fast, sweeps)
            if graph is not None:
                vals = graph.replay()                # one sync
                factors = graph.factors
            else:
                saved = list(factors)
                status = torch.zeros(order, dtype=torch.int32, device=t.device)
                core = _hooi_sweep(t, factors, fast, lambda y, r, warm: _factor_device(
                    y, r, ranks[r], warm, status, r, sweeps))
                vals = _hooi_status(core, status, torch.empty(
                    1 + order, dtype=torch.float64, device=t.device)).cpu().numpy()  # one sync
            stats["graph"] = graph is not None
            if np.all(vals[1:] == 1.0):
                norm_g = float(vals[0])
                stats["device_iterations"] += 1
            else:                                    # an unconverged factor: host path
                stats["host_redos"] += 1
                if graph is not None:
                    # the iteration's starting factors are intact in the
                    # other buffer set: redo on the host path, make the result
                    # the graph's current set
                    work = [f.clone() for f in graph.previous]
                    core = _hooi_sweep(t, work, fast, host_factor)
                    graph.load(work)
                    factors = graph.factors
                else:
                    factors[:] = saved
                    core = _hooi_sweep(t, factors, fast, host_factor)
                norm_g = _norm(core)
        else:
            core = _hooi_sweep(t, factors, fast, host_factor)
            norm_g = _norm(core)
            stats["host_iterations"] += 1
        resid = np.sqrt(max(0.0, norm_t ** 2 - norm_g ** 2))
        fit = 1.0 - resid / norm_t if norm_t > 0 else 1.0
        fits.append(fit)
        if fit - prev < tol and it > 0:
            break
        prev = fit
    # fresh tensors: graph-owned factors carry fp32 copies (_sbt_f32) that the
    # graph refreshes only on replay
    factors = [f.contiguous().clone() for f in factors]
    core = tucker_core(t, factors)
    return TuckerModel(core=core, factors=factors, fit_history=fits, iterations=iters,
                       stats=stats)
