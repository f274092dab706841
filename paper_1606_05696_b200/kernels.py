"""BLAS-like kernel API over flat device buffers (drop-in for sbtensor.kernels).

Entry points, argument meaning, validation and ``ValueError`` conditions
follow the reference (``/root/reference/pkg/src/sbtensor/kernels.py``):

* ``gemm``                    -- kernels.py:93-108
* ``strided_batched_gemm``    -- kernels.py:156-176
* ``strided_batched_gemm_ex`` -- kernels.py:207-225 (extended op flags EN/ET)
* ``strided_batched_gemm_ex_reference`` -- kernels.py:228-242 (per-batch loop)

Buffers are flat 1-D ``torch`` CUDA tensors (float32 or float64) and the work
is one launch of the sm_100a library on the current CUDA stream.  Flat numpy
arrays are also accepted: they take the library's host-buffer seam (copy in,
same kernels, copy out, synchronise) so reference-style callers run unchanged.
``threads`` is accepted for signature compatibility and ignored: the batch is
split across the GPU's SMs by the kernel's grid (reference kernels.py:245-266).

Beyond the reference checks (which guard the CPU loops), every call is also
bounds-checked against the buffer lengths, because an out-of-range stride on
the device would fault instead of raising.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from . import _lib


class Op(str, enum.Enum):
    Normal = "N"
    Transpose = "T"
    ExtendedNormal = "EN"
    ExtendedTranspose = "ET"


_PLAIN = (Op.Normal, Op.Transpose)
_EXTENDED = (Op.ExtendedNormal, Op.ExtendedTranspose)


@dataclass(frozen=True)
class KernelArgs:
    """Resolved argument block of one (possibly batched) kernel call
    (reference kernels.py:34-51)."""

    opa: Op
    opb: Op
    m: int
    n: int
    k: int
    alpha: float
    beta: float
    lda: int
    loa: int
    ldb: int
    lob: int
    ldc: int
    loc: int
    batch_count: int = 0


def _as_op(op) -> Op:
    if isinstance(op, Op):
        return op
    try:
        return Op(op)
    except ValueError:
        raise ValueError(f"unsupported op flag {op!r} (conjugate/Hermitian are rejected)") from None


def _op_strides(op: Op, rows: int, cols: int, ld: int, name: str):
    """Element (row, col) strides of op(X) for X stored column-major with
    leading dimension ld; ld must cover the stored rows (kernels.py:63-71)."""
    stored_rows = rows if op is Op.Normal else cols
    if ld < stored_rows:
        raise ValueError(f"{name}: leading dimension {ld} < stored rows {stored_rows}")
    return (1, ld) if op is Op.Normal else (ld, 1)


def _check_extents(m, n, k, batch_count=0):
    if min(m, n, k) < 1:
        raise ValueError(f"extents must be positive, got m={m} n={n} k={k}")
    if batch_count < 0:
        raise ValueError("batch_count must be non-negative")


def _check_c_regions(m, n, ldc, loc, batch_count):
    """C batch regions must provably not overlap: either interleaved
    (loc >= m and ldc >= loc*batch) or stacked (ldc >= m and loc >= n*ldc),
    the reference's conservative rule (kernels.py:81-90)."""
    if batch_count < 2:
        return
    if (loc >= m and ldc >= loc * batch_count) or (ldc >= m and loc >= n * ldc):
        return
    raise ValueError(
        f"overlapping C batch regions: m={m} n={n} ldc={ldc} loc={loc} batch={batch_count}")


def _check_ldc(m, ldc):
    if ldc < m:
        raise ValueError(f"C: leading dimension {ldc} < rows {m}")


# ---------------------------------------------------------------------------
# the one place every entry point lands: a fully strided (batched) core call

def _is_numpy(x):
    return isinstance(x, np.ndarray)


def _span(off, terms):
    return off + sum((e - 1) * s for e, s in terms if e > 0)


def _buffer_info(buf, name):
    if _is_numpy(buf):
        if buf.ndim != 1:
            raise ValueError(f"{name}: buffer must be a flat 1-D array")
        return buf.dtype, buf.size
    import torch
    if not isinstance(buf, torch.Tensor):
        raise TypeError(f"{name}: expected a torch tensor or numpy array, got {type(buf)!r}")
    if buf.dim() != 1 or not buf.is_contiguous():
        raise ValueError(f"{name}: buffer must be a contiguous 1-D tensor")
    if not buf.is_cuda:
        raise ValueError(f"{name}: torch buffers must live on a CUDA device")
    return buf.dtype, buf.numel()


def validate_call(m, n, k, a, oa, ars, acs, apt, b, ob, brs, bcs, bpt, c, oc, crs, ccs, cpt,
                  batch=1, apt2=0, bpt2=0, cpt2=0, batch2=1):
    """Buffer checks of one strided core call (every path into the library runs
    them: core_call and the grouped planner.execute_plans): flat contiguous
    buffers of one dtype on one side (host / device), non-negative strides, and
    every addressed element inside its buffer.  Returns (dtype, is_host)."""
    da, na = _buffer_info(a, "A")
    db, nb = _buffer_info(b, "B")
    dc, nc = _buffer_info(c, "C")
    host = _is_numpy(a)
    if _is_numpy(b) != host or _is_numpy(c) != host:
        raise ValueError("A, B and C must all be device tensors or all numpy arrays")
    if not (da == db == dc):
        raise ValueError(f"dtype mismatch: A {da}, B {db}, C {dc}")
    strides = (oa, ars, acs, apt, apt2, ob, brs, bcs, bpt, bpt2, oc, crs, ccs, cpt, cpt2)
    if min(strides) < 0:
        raise ValueError("offsets and strides must be non-negative")
    for name, top, size in (
            ("A", _span(oa, [(m, ars), (k, acs), (batch, apt), (batch2, apt2)]), na),
            ("B", _span(ob, [(k, brs), (n, bcs), (batch, bpt), (batch2, bpt2)]), nb),
            ("C", _span(oc, [(m, crs), (n, ccs), (batch, cpt), (batch2, cpt2)]), nc)):
        if top >= size:
            raise ValueError(f"{name}: call addresses element {top} of a buffer of {size}")
    return da, host


def core_call(m, n, k, alpha, a, oa, ars, acs, apt, b, ob, brs, bcs, bpt, beta, c, oc,
              crs, ccs, cpt, batch=1, apt2=0, bpt2=0, cpt2=0, batch2=1, extended=False):
    """Launch C = alpha*A.B + beta*C over strided views (the reference core
    signature, _loops_numba.py:12-35, plus an optional second batch mode)."""
    if batch == 0 or batch2 == 0:
        return
    da, host = validate_call(m, n, k, a, oa, ars, acs, apt, b, ob, brs, bcs, bpt, c, oc,
                             crs, ccs, cpt, batch, apt2, bpt2, cpt2, batch2)
    lib = _lib.load()
    if host:
        if str(da) not in ("float32", "float64"):
            raise ValueError(f"unsupported dtype {da}")
        f64 = str(da) == "float64"
        if batch2 != 1:
            for q in range(batch2):
                core_call(m, n, k, alpha, a, oa + q * apt2, ars, acs, apt, b, ob + q * bpt2,
                          brs, bcs, bpt, beta, c, oc + q * cpt2, crs, ccs, cpt, batch)
            return
        fn = lib.sbt_batched_core_host_f64 if f64 else lib.sbt_batched_core_host_f32
        for x in (a, b, c):
            if not x.flags.c_contiguous:
                raise ValueError("numpy buffers must be contiguous")
        if not c.flags.writeable:
            raise ValueError("C buffer is read-only")
        rc = fn(m, n, k, alpha, a.ctypes.data, oa, ars, acs, apt, b.ctypes.data, ob, brs, bcs,
                bpt, beta, c.ctypes.data, oc, crs, ccs, cpt, batch)
        _lib.check(rc, "strided batched GEMM (host buffers)")
        return
    import torch
    if da == torch.float64:
        f64 = True
    elif da == torch.float32:
        f64 = False
    else:
        raise ValueError(f"unsupported dtype {da}")
    if not (a.device == b.device == c.device):
        raise ValueError("A, B and C must be on the same device")
    dev = c.device.index
    if dev != torch.cuda.current_device():    # launch on C's device
        with torch.cuda.device(dev):
            return core_call(m, n, k, alpha, a, oa, ars, acs, apt, b, ob, brs, bcs, bpt, beta,
                             c, oc, crs, ccs, cpt, batch, apt2, bpt2, cpt2, batch2, extended)
    stream = torch.cuda.current_stream(dev).cuda_stream
    if True:
        if batch2 != 1:
            fn = lib.sbt_batched2_core_f64 if f64 else lib.sbt_batched2_core_f32
            rc = fn(m, n, k, alpha, a.data_ptr(), oa, ars, acs, apt, apt2, b.data_ptr(), ob,
                    brs, bcs, bpt, bpt2, beta, c.data_ptr(), oc, crs, ccs, cpt, cpt2, batch,
                    batch2, stream)
        else:
            if extended:
                fn = lib.sbt_ext_batched_core_f64 if f64 else lib.sbt_ext_batched_core_f32
            else:
                fn = lib.sbt_batched_core_f64 if f64 else lib.sbt_batched_core_f32
            rc = fn(m, n, k, alpha, a.data_ptr(), oa, ars, acs, apt, b.data_ptr(), ob, brs, bcs,
                    bpt, beta, c.data_ptr(), oc, crs, ccs, cpt, batch, stream)
    _lib.check(rc, "strided batched GEMM")


# ---------------------------------------------------------------------------
# reference entry points


def gemm(opa, opb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc,
         offa=0, offb=0, offc=0):
    """C = alpha * op(A) * op(B) + beta * C on column-major buffers; with
    beta == 0 the prior contents of C are never read (kernels.py:93-108)."""
    opa, opb = _as_op(opa), _as_op(opb)
    if opa not in _PLAIN or opb not in _PLAIN:
        raise ValueError("extended op flags are only accepted by strided_batched_gemm_ex")
    _check_extents(m, n, k)
    ars, acs = _op_strides(opa, m, k, lda, "A")
    brs, bcs = _op_strides(opb, k, n, ldb, "B")
    _check_ldc(m, ldc)
    core_call(m, n, k, alpha, a, offa, ars, acs, 0, b, offb, brs, bcs, 0, beta, c, offc,
              1, ldc, 0, batch=1)


def strided_batched_gemm(opa, opb, m, n, k, alpha, a, lda, loa, b, ldb, lob,
                         beta, c, ldc, loc, batch_count,
                         offa=0, offb=0, offc=0, threads=1):
    """batch_count GEMMs at constant strides loa/lob/loc between matrices, in
    one launch; lo = 0 broadcasts an operand (kernels.py:156-176)."""
    opa, opb = _as_op(opa), _as_op(opb)
    if opa not in _PLAIN or opb not in _PLAIN:
        raise ValueError("extended op flags are only accepted by strided_batched_gemm_ex")
    _check_extents(m, n, k, batch_count)
    if batch_count == 0:
        return
    ars, acs = _op_strides(opa, m, k, lda, "A")
    brs, bcs = _op_strides(opb, k, n, ldb, "B")
    _check_ldc(m, ldc)
    _check_c_regions(m, n, ldc, loc, batch_count)
    core_call(m, n, k, alpha, a, offa, ars, acs, loa, b, offb, brs, bcs, lob, beta, c, offc,
              1, ldc, loc, batch=batch_count)


def _extended_strides(opa, opb, m, n, k, lda, loa, ldb, lob):
    """(ars, acs, apt, brs, bcs, bpt) for the extended call: the extended
    operand is batched in its unit-stride first mode and (ld, lo) are the
    strides of its remaining two modes in storage order (kernels.py:179-204)."""
    a_ext, b_ext = opa in _EXTENDED, opb in _EXTENDED
    if a_ext == b_ext:
        raise ValueError("exactly one operand must carry an extended op flag")
    if a_ext:
        if opb not in _PLAIN:
            raise ValueError("non-extended operand must be Normal or Transpose")
        ars, acs = (lda, loa) if opa is Op.ExtendedNormal else (loa, lda)
        brs, bcs = _op_strides(opb, k, n, ldb, "B")
        return ars, acs, 1, brs, bcs, lob
    if opa not in _PLAIN:
        raise ValueError("non-extended operand must be Normal or Transpose")
    ars, acs = _op_strides(opa, m, k, lda, "A")
    brs, bcs = (ldb, lob) if opb is Op.ExtendedNormal else (lob, ldb)
    return ars, acs, loa, brs, bcs, 1


def strided_batched_gemm_ex(opa, opb, m, n, k, alpha, a, lda, loa, b, ldb, lob,
                            beta, c, ldc, loc, batch_count,
                            offa=0, offb=0, offc=0, threads=1):
    """Strided batched GEMM with one operand batched in its first stored mode,
    evaluated in place -- no permuted copy (kernels.py:207-225)."""
    opa, opb = _as_op(opa), _as_op(opb)
    _check_extents(m, n, k, batch_count)
    if batch_count == 0:
        return
    ars, acs, apt, brs, bcs, bpt = _extended_strides(opa, opb, m, n, k, lda, loa, ldb, lob)
    _check_ldc(m, ldc)
    _check_c_regions(m, n, ldc, loc, batch_count)
    core_call(m, n, k, alpha, a, offa, ars, acs, apt, b, offb, brs, bcs, bpt, beta, c, offc,
              1, ldc, loc, batch=batch_count, extended=True)


def strided_batched_gemm_ex_reference(opa, opb, m, n, k, alpha, a, lda, loa,
                                      b, ldb, lob, beta, c, ldc, loc, batch_count,
                                      offa=0, offb=0, offc=0):
    """Per-batch loop of single GEMM launches, for differential tests
    (kernels.py:228-242)."""
    opa, opb = _as_op(opa), _as_op(opb)
    _check_extents(m, n, k, batch_count)
    if batch_count == 0:
        return
    ars, acs, apt, brs, bcs, bpt = _extended_strides(opa, opb, m, n, k, lda, loa, ldb, lob)
    _check_c_regions(m, n, ldc, loc, batch_count)
    for p in range(batch_count):
        core_call(m, n, k, alpha, a, offa + p * apt, ars, acs, 0, b, offb + p * bpt, brs, bcs,
                  0, beta, c, offc + p * loc, 1, ldc, 0, batch=1)
