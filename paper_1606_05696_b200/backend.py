"""The reference's arithmetic seam, served by the B200 library.

``sbtensor.backend`` (reference ``backend.py:12-36``) selects a module that
exports ``gemm_core``, ``batched_core`` and ``ext_batched_core`` with the
signatures of ``_loops_numba.py:12-40`` over flat numpy buffers.  This module
exports exactly that table, implemented by the C ABI's host-buffer entry
points (copy the touched span to HBM, one sm_100a launch, copy C back,
synchronise), so the reference can select it as ``SBTENSOR_BACKEND=b200``
(see INTEGRATION.md).  ``blocked_core`` is out of scope (a CPU cache-tiling
experiment) and raises.
"""
from __future__ import annotations

import numpy as np

from . import _lib

BACKEND_NAME = "b200"


def _fn(buf, f64, f32):
    if buf.dtype == np.float64:
        return f64
    if buf.dtype == np.float32:
        return f32
    raise ValueError(f"unsupported buffer dtype {buf.dtype}")


def batched_core(m, n, k, alpha, a, oa, ars, acs, apt, b, ob, brs, bcs, bpt,
                 beta, c, oc, crs, ccs, cpt, batch):
    lib = _lib.load()
    fn = _fn(c, lib.sbt_batched_core_host_f64, lib.sbt_batched_core_host_f32)
    if not (a.dtype == b.dtype == c.dtype):
        raise ValueError("A, B and C must share a dtype")
    for x in (a, b, c):
        if x.ndim != 1 or not x.flags.c_contiguous:
            raise ValueError("buffers must be flat contiguous arrays")
    rc = fn(int(m), int(n), int(k), float(alpha), a.ctypes.data, int(oa), int(ars), int(acs),
            int(apt), b.ctypes.data, int(ob), int(brs), int(bcs), int(bpt), float(beta),
            c.ctypes.data, int(oc), int(crs), int(ccs), int(cpt), int(batch))
    _lib.check(rc, "batched_core")


ext_batched_core = batched_core


def gemm_core(m, n, k, alpha, a, oa, ars, acs, b, ob, brs, bcs, beta, c, oc, crs, ccs):
    batched_core(m, n, k, alpha, a, oa, ars, acs, 0, b, ob, brs, bcs, 0,
                 beta, c, oc, crs, ccs, 0, 1)


def blocked_core(*args, **kwargs):
    raise NotImplementedError("blocked_core (CPU cache-tile sweep) is not part of the B200 path")


def active_backend() -> str:
    return BACKEND_NAME
