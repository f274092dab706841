"""HOOI restatement (TEST INFRASTRUCTURE).

Follows ``tucker.hooi`` (``tucker.py:136-174``) step for step:

* init: factor r = leading left singular vectors of the mode-r unfolding via
  the Gram matrix ``mat @ mat.T`` (``tucker.py:63-76``), eigenvalues
  descending, each vector's largest-magnitude entry made positive;
* iterate: for r in modes, project T with every factor but r, transposed
  (``_mode_product_chain``, ``tucker.py:87-123``: modes with the larger
  reduction extent first, ties in ascending mode order), refresh factor r;
* fit = 1 - sqrt(max(0, ||T||^2 - ||G||^2)) / ||T||; stop when
  ``fit - prev < tol`` after the first iteration;
* core = T x_r U_r^T over all modes.

The only deviation is the eigensolver: the reference's cyclic Jacobi
(``tucker.py:21-60``, an n x n rotation matmul per pivot) is replaced by
``numpy.linalg.eigh`` (LAPACK), which is feasible at n=512.  Ordering and sign
conventions are identical, so factors agree up to the eigen-gap conditioning.
"""
from __future__ import annotations

import numpy as np


def unfold(arr: np.ndarray, r: int) -> np.ndarray:
    """Mode-r unfolding with the other modes in ascending order, column-major
    (``layout.py:218-230``)."""
    return np.moveaxis(arr, r, 0).reshape((arr.shape[r], -1), order="F")


def leading_left_singular_vectors(mat: np.ndarray, rank: int) -> np.ndarray:
    if rank > mat.shape[0]:
        raise ValueError(f"rank {rank} exceeds row count {mat.shape[0]}")
    gram = mat @ mat.T
    w, v = np.linalg.eigh(gram)
    order = np.argsort(w)[::-1]
    u = v[:, order[:rank]].copy()
    for j in range(rank):
        i = int(np.argmax(np.abs(u[:, j])))
        if u[i, j] < 0:
            u[:, j] = -u[:, j]
    return u


def mode_product(arr: np.ndarray, u: np.ndarray, r: int, transpose: bool) -> np.ndarray:
    """T x_r U^T (transpose=True, contracts dim_r) or T x_r U."""
    mat = u.T if transpose else u
    out = np.tensordot(mat, arr, axes=([1], [r]))
    return np.moveaxis(out, 0, r)


def mode_product_chain(arr, factors, skip, transpose):
    order = arr.ndim
    modes = [r for r in range(order) if r != skip]
    red = (lambda r: arr.shape[r]) if transpose else (lambda r: factors[r].shape[1])
    modes.sort(key=lambda r: -red(r))
    cur = arr
    for r in modes:
        cur = mode_product(cur, factors[r], r, transpose)
    return cur


def hooi(arr: np.ndarray, ranks, max_iters: int = 50, tol: float = 1e-10):
    arr = np.asarray(arr, np.float64)
    order = arr.ndim
    ranks = tuple(int(x) for x in ranks)
    if len(ranks) != order:
        raise ValueError(f"need {order} ranks, got {len(ranks)}")
    for r, (rank, dim) in enumerate(zip(ranks, arr.shape)):
        if not 1 <= rank <= dim:
            raise ValueError(f"rank {rank} invalid for mode {r} extent {dim}")
    factors = [leading_left_singular_vectors(unfold(arr, r), ranks[r]) for r in range(order)]
    norm_t = float(np.linalg.norm(arr))
    fits = []
    prev = -np.inf
    iters = 0
    for it in range(max_iters):
        iters = it + 1
        for r in range(order):
            y = mode_product_chain(arr, factors, r, True)
            factors[r] = leading_left_singular_vectors(unfold(y, r), ranks[r])
        core = mode_product_chain(arr, factors, None, True)
        norm_g = float(np.linalg.norm(core))
        resid = np.sqrt(max(0.0, norm_t ** 2 - norm_g ** 2))
        fit = 1.0 - resid / norm_t if norm_t > 0 else 1.0
        fits.append(fit)
        if fit - prev < tol and it > 0:
            break
        prev = fit
    core = mode_product_chain(arr, factors, None, True)
    return {"core": core, "factors": factors, "fit_history": fits, "iterations": iters}


def reconstruct(core, factors):
    return mode_product_chain(core, factors, None, False)
