"""numpy restatement of the reference arithmetic cores (TEST INFRASTRUCTURE).

Reference semantics restated here:

* ``gemm_core`` (``_loops_numba.py:12-25``): for every (i, j),
  ``acc = sum_l a[oa + i*ars + l*acs] * b[ob + l*brs + j*bcs]`` and
  ``c[oc + i*crs + j*ccs] = alpha*acc`` when ``beta == 0`` (C is never read),
  else ``alpha*acc + beta*c``.
* ``batched_core`` (``_loops_numba.py:28-35``): the same at offsets
  ``p*apt``, ``p*bpt``, ``p*cpt`` for p in [0, batch).  A zero batch stride
  broadcasts that operand (``test_kernels.py:84-96``).
* ``ext_batched_core`` (``_loops_numba.py:38-68``): identical arithmetic; the
  reference only changes the loop tiling.

All arithmetic is fp64 (the reference's ``acc = 0.0`` is a float64 even for
fp32 buffers), so fp32 device results are compared against an fp64 oracle run
on the same fp32 values upcast exactly.  Unlike the
reference numpy backend (``_loops_numpy.py:11`` hard-codes an 8-byte item size
and corrupts fp32 buffers) the views here use the buffer's own item size.
"""
from __future__ import annotations

import numpy as np


def _view(buf: np.ndarray, off: int, shape, strides, writeable=False):
    it = buf.itemsize
    return np.lib.stride_tricks.as_strided(
        buf[off:], shape=tuple(int(s) for s in shape),
        strides=tuple(int(s) * it for s in strides), writeable=writeable)


def _store(cv: np.ndarray, prod: np.ndarray, alpha: float, beta: float) -> None:
    if alpha != 1.0:
        prod *= alpha
    if beta == 0.0:
        cv[...] = prod
    else:
        cv[...] = prod + beta * np.asarray(cv, dtype=np.float64)


def _f64(v):
    return np.asarray(v, dtype=np.float64)


def gemm_core(m, n, k, alpha, a, oa, ars, acs, b, ob, brs, bcs, beta, c, oc, crs, ccs):
    av = _f64(_view(a, oa, (m, k), (ars, acs)))
    bv = _f64(_view(b, ob, (k, n), (brs, bcs)))
    cv = _view(c, oc, (m, n), (crs, ccs), writeable=True)
    _store(cv, av @ bv, float(alpha), float(beta))


def batched_core(m, n, k, alpha, a, oa, ars, acs, apt, b, ob, brs, bcs, bpt,
                 beta, c, oc, crs, ccs, cpt, batch):
    if batch <= 0:
        return
    if m * n * k >= 32768:
        # large matrices: the reference numpy backend's per-batch BLAS loop
        # (_loops_numpy.py:32-38) is the fastest host form
        for p in range(batch):
            gemm_core(m, n, k, alpha, a, oa + p * apt, ars, acs, b, ob + p * bpt, brs, bcs,
                      beta, c, oc + p * cpt, crs, ccs)
        return
    av = _f64(_view(a, oa, (batch, m, k), (apt, ars, acs)))
    bv = _f64(_view(b, ob, (batch, k, n), (bpt, brs, bcs)))
    cv = _view(c, oc, (batch, m, n), (cpt, crs, ccs), writeable=True)
    _store(cv, np.matmul(av, bv), float(alpha), float(beta))


ext_batched_core = batched_core


def batched2_core(m, n, k, alpha, a, oa, ars, acs, apt, apt2, b, ob, brs, bcs, bpt, bpt2,
                  beta, c, oc, crs, ccs, cpt, cpt2, batch, batch2):
    """Two nested batch modes = the reference's LoopStep loop around one
    batched call (``planner.py:551-581``)."""
    for q in range(batch2):
        batched_core(m, n, k, alpha, a, oa + q * apt2, ars, acs, apt,
                     b, ob + q * bpt2, brs, bcs, bpt,
                     beta, c, oc + q * cpt2, crs, ccs, cpt, batch)


def gemm_core_loops(m, n, k, alpha, a, oa, ars, acs, b, ob, brs, bcs, beta, c, oc, crs, ccs):
    """Element-by-element restatement (k ascending, one fp64 accumulator),
    for tiny extents where the exact reference loop order matters."""
    for j in range(n):
        for i in range(m):
            acc = 0.0
            for l in range(k):
                acc += float(a[oa + i * ars + l * acs]) * float(b[ob + l * brs + j * bcs])
            pc = oc + i * crs + j * ccs
            c[pc] = alpha * acc if beta == 0.0 else alpha * acc + beta * float(c[pc])
