"""Exhaustive-loop contraction oracle (TEST INFRASTRUCTURE).

Restates ``reference.contract_naive`` (``reference.py:27-51``): every output
element is one fp64 accumulator summed over the contracted indices in
ascending order; when ``beta == 0`` the prior C is never read.  Only feasible
at tiny extents; a vectorised fp64 ``einsum`` twin is provided for the
medium sizes the parity tests use.
"""
from __future__ import annotations

import itertools

import numpy as np


def _offset(labels, strides, env):
    return sum(env[l] * s for l, s in zip(labels, strides))


def contract_naive(la, lb, lc, ext, sa, sb, sc, a, b, alpha, beta, c):
    """Flat-buffer naive evaluation; ``s*`` are element strides per label."""
    kls = [l for l in la if l in lb]
    for out in itertools.product(*(range(ext[l]) for l in lc)):
        env = dict(zip(lc, out))
        acc = 0.0
        for kk in itertools.product(*(range(ext[l]) for l in kls)):
            env.update(zip(kls, kk))
            acc += float(a[_offset(la, sa, env)]) * float(b[_offset(lb, sb, env)])
        oc = _offset(lc, sc, env) if lc else 0
        prev = float(c[oc]) if beta != 0.0 else 0.0
        c[oc] = alpha * acc + beta * prev


def contract_einsum(la, lb, lc, a_arr, b_arr, alpha, beta, c_arr=None):
    """fp64 einsum on logical (multi-dimensional) arrays."""
    expr = f"{''.join(la)},{''.join(lb)}->{''.join(lc)}"
    out = alpha * np.einsum(expr, np.asarray(a_arr, np.float64), np.asarray(b_arr, np.float64),
                            optimize=True)
    if beta != 0.0 and c_arr is not None:
        out = out + beta * np.asarray(c_arr, np.float64)
    return out


def max_rel_err(got, want) -> float:
    """The reference's parity metric (``tests/conftest.py:31-35``)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    denom = float(np.max(np.abs(want))) if want.size else 0.0
    if denom == 0.0:
        return float(np.max(np.abs(got))) if got.size else 0.0
    return float(np.max(np.abs(got - want)) / denom)
