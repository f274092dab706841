"""Kernel-API lowering restated from ``kernels.py`` (TEST INFRASTRUCTURE).

``gemm`` / ``strided_batched_gemm`` / ``strided_batched_gemm_ex`` turn op flags
and leading dimensions into (row, col, batch) element strides before calling
a core: N -> (1, ld), T -> (ld, 1) (``kernels.py:63-71``); for the extended
operand EN -> (ld, lo), ET -> (lo, ld) with batch stride 1
(``kernels.py:179-204``); C is always (1, ldc, loc).
"""
from __future__ import annotations

from .cores import batched_core


def _plain(op, ld):
    return (1, ld) if op == "N" else (ld, 1)


def lower_call(fn, kw):
    """Map a reference kernel-API call (keyword form) to batched_core args."""
    opa, opb = kw["opa"], kw["opb"]
    m, n, k = kw["m"], kw["n"], kw["k"]
    if fn == "gemm":
        ars, acs = _plain(opa, kw["lda"])
        brs, bcs = _plain(opb, kw["ldb"])
        return dict(m=m, n=n, k=k, ars=ars, acs=acs, apt=0, brs=brs, bcs=bcs, bpt=0,
                    crs=1, ccs=kw["ldc"], cpt=0, batch=1,
                    oa=kw.get("offa", 0), ob=kw.get("offb", 0), oc=kw.get("offc", 0))
    batch = kw["batch_count"]
    if fn == "strided_batched_gemm":
        ars, acs = _plain(opa, kw["lda"])
        brs, bcs = _plain(opb, kw["ldb"])
        apt, bpt = kw["loa"], kw["lob"]
    elif fn == "strided_batched_gemm_ex":
        if opa in ("EN", "ET"):
            ars, acs = (kw["lda"], kw["loa"]) if opa == "EN" else (kw["loa"], kw["lda"])
            apt = 1
            brs, bcs = _plain(opb, kw["ldb"])
            bpt = kw["lob"]
        else:
            ars, acs = _plain(opa, kw["lda"])
            apt = kw["loa"]
            brs, bcs = (kw["ldb"], kw["lob"]) if opb == "EN" else (kw["lob"], kw["ldb"])
            bpt = 1
    else:
        raise ValueError(fn)
    return dict(m=m, n=n, k=k, ars=ars, acs=acs, apt=apt, brs=brs, bcs=bcs, bpt=bpt,
                crs=1, ccs=kw["ldc"], cpt=kw["loc"], batch=batch,
                oa=kw.get("offa", 0), ob=kw.get("offb", 0), oc=kw.get("offc", 0))


def run_call(fn, kw, a, b, c):
    cl = lower_call(fn, kw)
    batched_core(cl["m"], cl["n"], cl["k"], kw["alpha"], a, cl["oa"], cl["ars"], cl["acs"],
                 cl["apt"], b, cl["ob"], cl["brs"], cl["bcs"], cl["bpt"], kw["beta"], c,
                 cl["oc"], cl["crs"], cl["ccs"], cl["cpt"], cl["batch"])
