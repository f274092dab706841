"""Restatement of the reference single-mode dispatcher (TEST INFRASTRUCTURE).

``lower(labels_a, labels_b, labels_c, dims/strides...)`` follows
``planner.plan_single_mode`` (``planner.py:218-371``) and
``planner._execute_batched`` (``planner.py:508-581``) and returns

* ``strategy``   -- flattened-gemm | strided-batched | nested-batched |
                    extended-batched (the reference's names);
* ``args``       -- the reference's ``resolved_kernel_args`` fields
                    (``planner.py:784-830``): opa, opb, m, n, k, lda, loa, ldb,
                    lob, ldc, loc, batch_count;
* ``calls``      -- every arithmetic-core call the reference issues, already
                    lowered to the core's stride form (``kernels.py:63-71``,
                    ``:179-204``): one dict per call with the ``batched_core``
                    argument names plus ``first`` ("A"/"B": which tensor sits in
                    the kernel's A slot).

It is written independently of the product planner so the two can be
cross-checked against each other and against tests/golden/plans.json.
"""
from __future__ import annotations

import itertools
from math import prod


class OraclePlanError(ValueError):
    pass


def _modes(labels, dims, strides):
    return [[l, int(d), int(s)] for l, d, s in zip(labels, dims, strides)]


def _pos(modes, label):
    for i, md in enumerate(modes):
        if md[0] == label:
            return i
    return -1


def _stride(modes, label):
    i = _pos(modes, label)
    return None if i < 0 else modes[i][2]


def lower(la, lb, lc, dims_a, strides_a, dims_b, strides_b, dims_c, strides_c):
    la, lb, lc = tuple(la), tuple(lb), tuple(lc)
    kset = [l for l in la if l in lb]
    if len(kset) != 1:
        raise OraclePlanError("exactly one contracted index required")
    kl = kset[0]
    A = _modes(la, dims_a, strides_a)
    B = _modes(lb, dims_b, strides_b)
    C = _modes(lc, dims_c, strides_c) if lc else []
    ext = {md[0]: md[1] for md in A + B}
    # squeeze extent-1 free modes (planner.py:247-250)
    A = [md for md in A if md[0] == kl or md[1] > 1]
    B = [md for md in B if md[0] == kl or md[1] > 1]
    C = [md for md in C if md[1] > 1]
    T = {"A": A, "B": B, "C": C}
    owner = {md[0]: "A" for md in A if md[0] != kl}
    owner.update({md[0]: "B" for md in B if md[0] != kl})
    # greedy flattening of output runs (planner.py:252-285)
    i = 0
    while i < len(T["C"]) - 1:
        c = T["C"]
        o = owner[c[i][0]]
        src = T[o]
        j = i
        while j + 1 < len(c) and owner.get(c[j + 1][0]) == o:
            p = _pos(src, c[j][0])
            if p < 0 or p + 1 >= len(src) or src[p + 1][0] != c[j + 1][0]:
                break
            if c[j + 1][2] != c[j][2] * c[j][1] or src[p + 1][2] != src[p][2] * src[p][1]:
                break
            j += 1
        if j > i:
            run = [md[0] for md in c[i:j + 1]]
            name = "".join(run)
            for t in (o, "C"):
                lst = T[t]
                p = _pos(lst, run[0])
                grp = lst[p:p + len(run)]
                lst[p:p + len(run)] = [[name, prod(g[1] for g in grp), grp[0][2]]]
            owner[name] = o
            ext[name] = prod(ext[r] for r in run)
        i += 1
    A, B, C = T["A"], T["B"], T["C"]
    cpos = {md[0]: idx for idx, md in enumerate(C)}

    if not C:
        # scalar output: DOT via gemm(N, N, 1, 1, k)
        x, y = A, B
        lda = _stride(x, kl)
        return _finish("flattened-gemm", "A", "N", "N", 1, 1, ext[kl], x, y, C,
                       lda, 0, ext[kl], 0, 1, 0, 0, None, [], False, kl, None, None)
    if C[0][2] != 1:
        raise OraclePlanError("output's leading free mode must have unit stride")
    c1 = C[0][0]
    first = "A" if _pos(A, c1) >= 0 else "B"
    X, Y = (A, B) if first == "A" else (B, A)
    fx = [md for md in X if md[0] not in (c1, kl)]
    fy = [md for md in Y if md[0] != kl]
    nmode = None
    if fy:
        nmode = Y[0] if Y[0][0] != kl else max(fy, key=lambda md: (md[1], cpos[md[0]]))
    op2 = "N" if (nmode is None or Y[0][0] == kl) else "T"
    rest = fx + [md for md in fy if nmode is None or md[0] != nmode[0]]
    m = ext[c1]
    n = nmode[1] if nmode else 1
    k = ext[kl]
    ldb = (_stride(Y, nmode[0]) if nmode else k) if op2 == "N" else _stride(Y, kl)
    ldc = _stride(C, nmode[0]) if nmode else max(m, 1)
    if X[0][0] not in (c1, kl):
        batch = X[0]
        rest = [md for md in rest if md[0] != batch[0]]
        op1 = "EN" if _pos(X, c1) < _pos(X, kl) else "ET"
        two = [md for md in X if md[0] in (c1, kl)]
        lda, loa = two[0][2], two[1][2]
        loops = sorted(rest, key=lambda md: cpos[md[0]])
        lob = _stride(Y, batch[0]) or 0
        return _finish("extended-batched", first, op1, op2, m, n, k, X, Y, C,
                       lda, loa, ldb, lob, ldc, _stride(C, batch[0]), batch[1], batch,
                       loops, True, kl, c1, nmode)
    op1 = "N" if X[0][0] == c1 else "T"
    lda = _stride(X, kl) if op1 == "N" else _stride(X, c1)
    if not rest:
        return _finish("flattened-gemm", first, op1, op2, m, n, k, X, Y, C,
                       lda, 0, ldb, 0, ldc, 0, 0, None, [], False, kl, c1, nmode)
    batch = max(rest, key=lambda md: (md[1], cpos[md[0]]))
    loops = sorted([md for md in rest if md[0] != batch[0]], key=lambda md: cpos[md[0]])
    return _finish("nested-batched" if loops else "strided-batched", first, op1, op2,
                   m, n, k, X, Y, C, lda, _stride(X, batch[0]) or 0, ldb,
                   _stride(Y, batch[0]) or 0, ldc, _stride(C, batch[0]), batch[1], batch,
                   loops, False, kl, c1, nmode)


def _plain(op, ld):
    return (1, ld) if op == "N" else (ld, 1)


def _finish(strategy, first, op1, op2, m, n, k, X, Y, C, lda, loa, ldb, lob, ldc, loc,
            batch_count, batch, loops, extended, kl, c1, nmode):
    args = dict(opa=op1, opb=op2, m=m, n=n, k=k, lda=lda or max(m, 1), loa=loa,
                ldb=ldb or k, lob=lob, ldc=ldc or max(m, 1), loc=loc if batch else 0,
                batch_count=batch_count if batch else 0)
    if extended:
        ars, acs = (lda, loa) if op1 == "EN" else (loa, lda)
        apt = 1
    else:
        ars, acs = _plain(op1, lda)
        apt = loa
    brs, bcs = _plain(op2, ldb)
    base = dict(m=m, n=n, k=k, ars=ars, acs=acs, apt=apt, brs=brs, bcs=bcs, bpt=lob,
                crs=1, ccs=ldc, cpt=loc if batch else 0,
                batch=batch_count if batch else 1, first=first)
    if not batch:
        base.update(apt=0, bpt=0, cpt=0)
    calls = []
    A_, B_ = ("A", "B") if first == "A" else ("B", "A")
    for combo in itertools.product(*(range(md[1]) for md in loops)):
        off = {"X": 0, "Y": 0, "C": 0}
        for md, idx in zip(loops, combo):
            for name, lst in (("X", X), ("Y", Y), ("C", C)):
                s = _stride(lst, md[0])
                if s is not None:
                    off[name] += idx * s
        calls.append(dict(base, oa=off["X"], ob=off["Y"], oc=off["C"]))
    return {"strategy": strategy, "first": first, "args": args, "calls": calls,
            "loops": [[md[0], md[1]] for md in loops],
            "batch_label": batch[0] if batch else None, "extended": extended}


def execute(lowered, a, b, alpha, beta, c, core=None):
    """Run every lowered core call on flat numpy buffers (C mutated in place)."""
    from .cores import batched_core
    core = core or batched_core
    x, y = (a, b) if lowered["first"] == "A" else (b, a)
    for cl in lowered["calls"]:
        core(cl["m"], cl["n"], cl["k"], alpha, x, cl["oa"], cl["ars"], cl["acs"], cl["apt"],
             y, cl["ob"], cl["brs"], cl["bcs"], cl["bpt"], beta, c, cl["oc"], cl["crs"],
             cl["ccs"], cl["cpt"], cl["batch"])


def packed_strides(dims):
    out, s = [], 1
    for d in dims:
        out.append(s)
        s *= d
    return out


def contract(labels_a, labels_b, labels_c, ext, a, b, alpha, beta, c, layouts=None):
    """Plan + execute a contraction exactly as the reference would (packed
    operands, or the (dims, strides) of ``layouts`` = (la, lb, lc))."""
    da = [ext[l] for l in labels_a]
    db = [ext[l] for l in labels_b]
    dc = [ext[l] for l in labels_c] or [1]
    if layouts is None:
        sa, sb, sc = packed_strides(da), packed_strides(db), packed_strides(dc)
    else:
        sa, sb, sc = (list(x.strides) for x in layouts)
    low = lower(labels_a, labels_b, labels_c, da, sa, db, sb, dc, sc)
    execute(low, a, b, alpha, beta, c)
    return low
