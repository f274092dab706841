"""Comparison evaluators (reference reference.py:19-63).

``contract_conventional`` runs the permute-then-GEMM strategy on the device --
the baseline the paper's transpose-free SBGEMM is measured against
(Fig. 1/4).  The naive loop evaluator ``contract_naive`` is the
reference's ground truth and lives in ``oracle/naive.py`` (test
infrastructure), not in this package.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

from .layout import DenseTensor
from .notation import ContractionSpec
from .planner import execute_plan, plan_conventional


@dataclass
class EvalCounters:
    """Copy / transposition / launch counters of one evaluation
    (reference reference.py:19-24)."""
    transpositions: int = 0
    bytes_copied: int = 0
    kernel_calls: dict = field(default_factory=dict)
    elapsed: float = 0.0


def contract_conventional(spec: ContractionSpec, a: DenseTensor, b: DenseTensor,
                          alpha: float, beta: float, c: DenseTensor,
                          policy: str = "opt") -> EvalCounters:
    """Matricized (permute, GEMM, permute back) evaluation on the device;
    returns the copy / transposition counters (reference reference.py:54-63).
    ``elapsed`` is host wall time including a device synchronisation."""
    import torch
    plan = plan_conventional(spec, a.layout, b.layout, c.layout, policy=policy)
    counters = EvalCounters()
    t0 = time.perf_counter()
    execute_plan(plan, a, b, alpha, beta, c, counters=counters)
    torch.cuda.synchronize(c.data.device)
    counters.elapsed = time.perf_counter() - t0
    return counters
