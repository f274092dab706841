"""Single-mode contraction planning onto transpose-free strided batched GEMM.

Planning semantics are the reference's (``planner.py:218-371``), so every
case gets the same strategy, operand roles, op flags, batch mode and loop
modes:

1. extent-1 free modes are squeezed away;
2. maximal runs of output modes that are contiguous and stride-mergeable in
   both C and their owning operand are flattened into one GEMM mode;
3. the operand owning C's first (unit-stride) mode provides the GEMM rows;
   the other operand's GEMM column mode is its first stored mode when that is
   free, else its largest free mode (ties -> later in C);
4. if the first operand's unit-stride mode is neither C's first mode nor the
   contracted one, the plan is the *extended* (exceptional) form, batched in
   that unit-stride mode; otherwise the largest remaining free mode (ties ->
   later in C) is the batch mode and any others become loop modes.

Execution is where this build departs: ``execute_plan`` lowers the plan to
ONE launch of the sm_100a library -- the batch mode and the innermost loop
mode become the kernel's two grid batch dimensions (the reference runs a
Python loop of batched calls, ``planner.py:551-581``) -- using the operands'
actual element strides, so no operand is ever copied or permuted.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from math import factorial, prod

from .kernels import KernelArgs, Op, core_call
from .layout import DenseTensor, Layout, permute_copy, permute_into
from .notation import ContractionSpec, classify_indices, kernel_family


class PlanError(ValueError):
    pass


class UnsupportedContractionError(PlanError):
    """The single-mode planner requires exactly one contracted index."""


class PlanConsistencyError(PlanError):
    """Tensors passed to execute_plan do not match the planned layouts."""


_FREE_LETTERS = "mnpqrstuvw"


@dataclass(frozen=True)
class Mode:
    label: str
    extent: int
    stride: int


@dataclass(frozen=True)
class FlattenStep:
    tensor: str
    labels: tuple
    merged: str


@dataclass(frozen=True)
class LoopStep:
    label: str
    extent: int


@dataclass(frozen=True)
class GemmStep:
    first: str                  # tensor providing GEMM rows: "A" | "B"
    op_first: Op
    op_second: Op
    m_label: object
    n_label: object
    k_label: str


@dataclass(frozen=True)
class BatchedStep:
    gemm: GemmStep
    batch_label: str
    extent: int
    extended: bool = False


@dataclass(frozen=True)
class GemvBatchStep:
    loop_labels: tuple
    matrix: str                 # tensor acting as the GEMV matrix
    op: Op
    v_label: str                # output mode of each GEMV
    k_label: str


@dataclass(frozen=True)
class PermuteStep:
    tensor: str
    perm: tuple


@dataclass(frozen=True)
class ConventionalInfo:
    free_a: tuple
    free_b: tuple
    contracted: tuple
    op_a: Op
    op_b: Op
    permute_a: object           # tuple | None
    permute_b: object
    c_matches: bool             # C's label order is already free_a + free_b
    family: str
    policy: str


@dataclass
class EvaluationPlan:
    spec: ContractionSpec
    layout_a: Layout
    layout_b: Layout
    layout_c: Layout
    strategy: str
    steps: list = field(default_factory=list)
    predicted_transpositions: int = 0
    eff: dict = field(default_factory=dict)
    conventional: object = None
    _launch: object = field(default=None, repr=False, compare=False)


@dataclass(frozen=True)
class CaseDescriptor:
    case_id: str
    labels_a: tuple
    labels_b: tuple
    labels_c: tuple
    classification: str         # single-gemm | strided-batched | exceptional


# ---------------------------------------------------------------------------
# the 36-case (and general (a, b)-order) catalogue


def _insert(seq, pos, item):
    out = list(seq)
    out.insert(pos, item)
    return tuple(out)


def enumerate_cases(order_a: int, order_b: int) -> list:
    """Every single-mode contraction pattern of an order-a by order-b pair with
    C fixed as the free labels in order; (a+b-2)! * a * b cases.  Case ids are
    "<family>.<variant>": families enumerate A's free labels (permutations) and
    k's position in A from the back; variants enumerate k's position in B then
    B's free-label permutations (reference planner.py:132-167)."""
    if order_a < 1 or order_b < 1:
        raise ValueError("orders must be >= 1")
    n_free = order_a + order_b - 2
    if n_free > len(_FREE_LETTERS):
        raise ValueError("orders too large to label")
    free = tuple(_FREE_LETTERS[:n_free])
    families = [(a_free, kpos) for a_free in itertools.permutations(free, order_a - 1)
                for kpos in reversed(range(order_a))]
    cases = []
    for fam, (a_free, kpos_a) in enumerate(families, start=1):
        labels_a = _insert(a_free, kpos_a, "k")
        others = [l for l in free if l not in a_free]
        variants = [_insert(b_free, kpos_b, "k") for kpos_b in range(order_b)
                    for b_free in itertools.permutations(others)]
        for var, labels_b in enumerate(variants, start=1):
            spec = ContractionSpec(labels_a, labels_b, free)
            cases.append(CaseDescriptor(f"{fam}.{var}", labels_a, labels_b, free,
                                        _classify(spec)))
    assert len(cases) == factorial(n_free) * order_a * order_b
    return cases


def find_case(order_a: int, order_b: int, case_id: str) -> CaseDescriptor:
    for case in enumerate_cases(order_a, order_b):
        if case.case_id == case_id:
            return case
    raise PlanError(f"no case {case_id} for orders ({order_a}, {order_b})")


def _classify(spec: ContractionSpec) -> str:
    """Structural class at packed layouts with distinct extents 3, 4, ... per
    (sorted) label (reference planner.py:177-194)."""
    labels = sorted(set(spec.labels_a) | set(spec.labels_b))
    ext = {l: 3 + i for i, l in enumerate(labels)}
    lay = [Layout.packed([ext[l] for l in labs] or [1])
           for labs in (spec.labels_a, spec.labels_b, spec.labels_c)]
    strategy = plan_single_mode(spec, *lay).strategy
    return {"flattened-gemm": "single-gemm",
            "extended-batched": "exceptional"}.get(strategy, "strided-batched")


def classify_case(case: CaseDescriptor) -> str:
    return case.classification


# ---------------------------------------------------------------------------
# planning


class _ModeList(list):
    def index_of(self, label):
        for i, md in enumerate(self):
            if md.label == label:
                return i
        return -1

    def stride(self, label):
        i = self.index_of(label)
        return None if i < 0 else self[i].stride


def _modes(labels, layout):
    if len(labels) != layout.order:
        raise PlanError(f"{len(labels)} labels for order-{layout.order} layout")
    return _ModeList(Mode(l, d, s) for l, d, s in zip(labels, layout.dims, layout.strides))


def _merge_runs(plan, tensors, owner):
    """Greedy flattening of output runs (reference planner.py:252-285)."""
    pos = 0
    while pos < len(tensors["C"]) - 1:
        out = tensors["C"]
        who = owner[out[pos].label]
        src = tensors[who]
        end = pos
        while end + 1 < len(out) and owner.get(out[end + 1].label) == who:
            at = src.index_of(out[end].label)
            nxt = out[end + 1]
            if at < 0 or at + 1 >= len(src) or src[at + 1].label != nxt.label:
                break
            if nxt.stride != out[end].stride * out[end].extent:
                break
            if src[at + 1].stride != src[at].stride * src[at].extent:
                break
            end += 1
        if end > pos:
            run = tuple(md.label for md in out[pos:end + 1])
            merged = "".join(run)
            for t in (who, "C"):
                lst = tensors[t]
                at = lst.index_of(run[0])
                group = lst[at:at + len(run)]
                lst[at:at + len(run)] = [Mode(merged, prod(g.extent for g in group),
                                              group[0].stride)]
                plan.steps.append(FlattenStep(t, run, merged))
            owner[merged] = who
        pos += 1


def plan_single_mode(spec: ContractionSpec, layout_a: Layout, layout_b: Layout,
                     layout_c: Layout) -> EvaluationPlan:
    contracted = classify_indices(spec).contracted
    if len(contracted) != 1:
        raise UnsupportedContractionError(
            f"single-mode planner requires exactly one contracted index, got {contracted}")
    k = contracted[0]
    A = _modes(spec.labels_a, layout_a)
    B = _modes(spec.labels_b, layout_b)
    if spec.labels_c:
        C = _modes(spec.labels_c, layout_c)
    else:
        if layout_c.dims != (1,):
            raise PlanError("scalar output requires a single-element layout")
        C = _ModeList()
    extent = {md.label: md.extent for md in (*A, *B)}
    for md in C:
        if extent.get(md.label) != md.extent:
            raise PlanError(f"extent mismatch for output label {md.label!r}")
    if A[A.index_of(k)].extent != B[B.index_of(k)].extent:
        raise PlanError(f"extent mismatch for contracted label {k!r}")

    plan = EvaluationPlan(spec=spec, layout_a=layout_a, layout_b=layout_b,
                          layout_c=layout_c, strategy="", steps=[])
    keep = lambda md: md.label == k or md.extent > 1  # noqa: E731
    tensors = {"A": _ModeList(filter(keep, A)), "B": _ModeList(filter(keep, B)),
               "C": _ModeList(md for md in C if md.extent > 1)}
    owner = {md.label: "A" for md in tensors["A"]}
    owner.update({md.label: "B" for md in tensors["B"] if md.label != k})
    _merge_runs(plan, tensors, owner)
    A, B, C = tensors["A"], tensors["B"], tensors["C"]
    plan.eff = {"A": tuple(A), "B": tuple(B), "C": tuple(C)}

    if not C:
        plan.steps.append(GemmStep("A", Op.Normal, Op.Normal, None, None, k))
        plan.strategy = "flattened-gemm"
        return plan
    if C[0].stride != 1:
        raise PlanError("output's leading free mode must have unit stride")
    c1 = C[0].label
    first = "A" if A.index_of(c1) >= 0 else "B"
    X, Y = (A, B) if first == "A" else (B, A)
    c_rank = lambda md: C.index_of(md.label)  # noqa: E731
    free_x = [md for md in X if md.label not in (c1, k)]
    free_y = [md for md in Y if md.label != k]
    n_mode = None
    if free_y:
        n_mode = Y[0] if Y[0].label != k else max(free_y, key=lambda md: (md.extent, c_rank(md)))
    op_second = Op.Normal if (n_mode is None or Y[0].label == k) else Op.Transpose
    rest = free_x + [md for md in free_y if n_mode is None or md.label != n_mode.label]
    n_label = n_mode.label if n_mode else None

    if X[0].label not in (c1, k):
        batch = X[0]
        rest = [md for md in rest if md.label != batch.label]
        op_first = (Op.ExtendedNormal if X.index_of(c1) < X.index_of(k)
                    else Op.ExtendedTranspose)
        for md in sorted(rest, key=c_rank):
            plan.steps.append(LoopStep(md.label, md.extent))
        plan.steps.append(BatchedStep(GemmStep(first, op_first, op_second, c1, n_label, k),
                                      batch.label, batch.extent, extended=True))
        plan.strategy = "extended-batched"
        return plan

    op_first = Op.Normal if X[0].label == c1 else Op.Transpose
    gemm = GemmStep(first, op_first, op_second, c1, n_label, k)
    if not rest:
        plan.steps.append(gemm)
        plan.strategy = "flattened-gemm"
        return plan
    batch = max(rest, key=lambda md: (md.extent, c_rank(md)))
    loops = sorted((md for md in rest if md.label != batch.label), key=c_rank)
    for md in loops:
        plan.steps.append(LoopStep(md.label, md.extent))
    plan.steps.append(BatchedStep(gemm, batch.label, batch.extent))
    plan.strategy = "nested-batched" if loops else "strided-batched"
    return plan


# ---------------------------------------------------------------------------
# lowering and execution


@dataclass(frozen=True)
class Launch:
    """One library launch (plus the outer loop combos for plans with more than
    one loop mode) with element strides taken from the planned layouts."""

    first: str
    m: int
    n: int
    k: int
    strides: tuple              # (ars, acs, apt, apt2, brs, bcs, bpt, bpt2, crs, ccs, cpt, cpt2)
    batch: int
    batch2: int
    outer: tuple                # ((x_off, y_off, c_off), ...) for loops beyond the fused one
    extended: bool
    kind: str


def _gemm_and_batch(plan):
    last = plan.steps[-1] if plan.steps else None
    if isinstance(last, BatchedStep):
        return last.gemm, last
    if isinstance(last, GemmStep):
        return last, None
    raise PlanError(f"plan strategy {plan.strategy!r} has no GEMM step")


def lower_plan(plan: EvaluationPlan) -> Launch:
    if plan._launch is not None:
        return plan._launch
    gemm, batch = _gemm_and_batch(plan)
    eff = {t: _ModeList(plan.eff[t]) for t in "ABC"}
    X, Y = (eff["A"], eff["B"]) if gemm.first == "A" else (eff["B"], eff["A"])
    C = eff["C"]
    ext = {md.label: md.extent for md in (*eff["A"], *eff["B"], *C)}

    def st(lst, label):
        return (lst.stride(label) or 0) if label is not None else 0

    m = ext[gemm.m_label] if gemm.m_label else 1
    n = ext[gemm.n_label] if gemm.n_label else 1
    k = ext[gemm.k_label]
    ars, acs = st(X, gemm.m_label), st(X, gemm.k_label)
    brs, bcs = st(Y, gemm.k_label), st(Y, gemm.n_label)
    crs, ccs = st(C, gemm.m_label), st(C, gemm.n_label)
    nb, apt, bpt, cpt = 1, 0, 0, 0
    if batch is not None:
        nb = batch.extent
        apt, bpt, cpt = st(X, batch.batch_label), st(Y, batch.batch_label), st(C, batch.batch_label)
    loops = [s for s in plan.steps if isinstance(s, LoopStep)]
    nb2, apt2, bpt2, cpt2 = 1, 0, 0, 0
    if loops:
        inner = loops[-1]
        nb2 = inner.extent
        apt2, bpt2, cpt2 = st(X, inner.label), st(Y, inner.label), st(C, inner.label)
    outer = []
    for combo in itertools.product(*(range(s.extent) for s in loops[:-1])):
        offs = [0, 0, 0]
        for s, idx in zip(loops[:-1], combo):
            for t, lst in enumerate((X, Y, C)):
                offs[t] += idx * st(lst, s.label)
        outer.append(tuple(offs))
    kind = ("gemm" if batch is None else
            "strided_batched_gemm_ex" if batch.extended else "strided_batched_gemm")
    plan._launch = Launch(gemm.first, m, n, k,
                          (ars, acs, apt, apt2, brs, bcs, bpt, bpt2, crs, ccs, cpt, cpt2),
                          nb, nb2, tuple(outer) or ((0, 0, 0),),
                          bool(batch is not None and batch.extended), kind)
    return plan._launch


# ---------------------------------------------------------------------------
# the conventional comparison strategy (reference planner.py:411-465, 620-713)


def plan_conventional(spec: ContractionSpec, layout_a: Layout, layout_b: Layout,
                      layout_c: Layout, policy: str = "opt") -> EvaluationPlan:
    """Permute-and-matricize plan: bring operands to C_IJ = A_IK B_KJ form
    (reference planner.py:411-465, same steps and transposition count).

    policy "opt" replaces single leading-block swaps with transpose op flags
    and skips the output pre-permute when beta == 0; "naive" materializes
    every permutation.  This is the baseline the paper measures SBGEMM
    against; execute_plan runs it on the device (permute kernel + one GEMM)."""
    if policy not in ("opt", "naive"):
        raise PlanError(f"unknown conventional policy {policy!r}")
    cls = classify_indices(spec)
    plan = EvaluationPlan(spec=spec, layout_a=layout_a, layout_b=layout_b,
                          layout_c=layout_c, strategy="conventional", steps=[])
    _modes(spec.labels_a, layout_a)
    _modes(spec.labels_b, layout_b)
    if spec.labels_c:
        _modes(spec.labels_c, layout_c)
    for name, lay in (("A", layout_a), ("B", layout_b), ("C", layout_c)):
        if not lay.is_packed():
            raise PlanError(f"conventional evaluation requires packed {name}")
    target_a = cls.free_a + cls.contracted
    target_b = cls.contracted + cls.free_b
    op_a = op_b = Op.Normal
    perm_a = perm_b = None
    if spec.labels_a != target_a:
        if policy == "opt" and spec.labels_a == cls.contracted + cls.free_a:
            op_a = Op.Transpose
        else:
            perm_a = tuple(spec.labels_a.index(l) for l in target_a)
            plan.steps.append(PermuteStep("A", perm_a))
    if spec.labels_b != target_b:
        if policy == "opt" and spec.labels_b == cls.free_b + cls.contracted:
            op_b = Op.Transpose
        else:
            perm_b = tuple(spec.labels_b.index(l) for l in target_b)
            plan.steps.append(PermuteStep("B", perm_b))
    target_c = cls.free_a + cls.free_b
    c_matches = spec.labels_c == target_c
    if not c_matches:
        if policy == "naive" or spec.beta != 0.0:
            plan.steps.append(PermuteStep("C", tuple(spec.labels_c.index(l) for l in target_c)))
        plan.steps.append(PermuteStep("C", tuple(target_c.index(l) for l in spec.labels_c)))
    plan.conventional = ConventionalInfo(
        free_a=cls.free_a, free_b=cls.free_b, contracted=cls.contracted, op_a=op_a, op_b=op_b,
        permute_a=perm_a, permute_b=perm_b, c_matches=c_matches, family=kernel_family(cls),
        policy=policy)
    plan.predicted_transpositions = sum(1 for st in plan.steps if isinstance(st, PermuteStep))
    return plan


def _eff_find(eff, label):
    for i, mode in enumerate(eff):
        if mode.label == label:
            return i
    return -1


def _eff_stride(eff, label):
    i = _eff_find(eff, label)
    return eff[i].stride if i >= 0 else None


def plan_batched_gemv(spec: ContractionSpec, layout_a: Layout, layout_b: Layout,
                      layout_c: Layout) -> EvaluationPlan:
    """Looped-GEMV evaluation (reference planner.py:374-404): no copies, lower
    arithmetic intensity -- the third strategy of the paper's exceptional-case
    comparison (Fig. 10).  Executed on the device as ONE batched
    GEMV launch (loop modes become the grid's batch modes)."""
    cls = classify_indices(spec)
    if len(cls.contracted) != 1:
        raise UnsupportedContractionError("batched-gemv planning is single-mode only")
    k_label = cls.contracted[0]
    plan = plan_single_mode(spec, layout_a, layout_b, layout_c)  # squeeze / flatten
    ea, eb, ec = plan.eff["A"], plan.eff["B"], plan.eff["C"]
    if not ec:
        raise PlanError("scalar output has no batched-gemv form")
    c1 = ec[0].label
    first = "A" if _eff_find(ea, c1) >= 0 else "B"
    ex = ea if first == "A" else eb
    if ex[0].label == k_label:
        v_label, op = c1, Op.Transpose
    elif ex[0].label == c1:
        v_label, op = c1, Op.Normal
    else:
        v_label, op = ex[0].label, Op.Normal
    loops = tuple(m.label for m in ec if m.label != v_label)
    gplan = EvaluationPlan(spec=spec, layout_a=layout_a, layout_b=layout_b,
                           layout_c=layout_c, strategy="batched-gemv",
                           steps=[st for st in plan.steps if isinstance(st, FlattenStep)],
                           eff=plan.eff)
    gplan.steps.append(GemvBatchStep(loop_labels=loops, matrix=first, op=op,
                                     v_label=v_label, k_label=k_label))
    return gplan


def _execute_gemv(plan, a, b, alpha, beta, c, counters):
    """Device execution of a batched-GEMV plan: every GEMV of the reference's
    loop (planner.py:584-617) in one strided batched launch with n = 1."""
    eff = plan.eff
    ea, eb, ec = eff["A"], eff["B"], eff["C"]
    st = plan.steps[-1]
    ex, ey = (ea, eb) if st.matrix == "A" else (eb, ea)
    bx, by = (a, b) if st.matrix == "A" else (b, a)
    extent = {mo.label: mo.extent for mo in (*ea, *eb, *ec)}
    # y[v] = sum_k X[v, k] x[k]  (op only records which X mode is unit stride)
    m, kk = extent[st.v_label], extent[st.k_label]
    ars, acs = _eff_stride(ex, st.v_label), _eff_stride(ex, st.k_label)
    brs, crs = _eff_stride(ey, st.k_label), _eff_stride(ec, st.v_label)
    loops = [(extent[l], _eff_stride(ex, l) or 0, _eff_stride(ey, l) or 0,
              _eff_stride(ec, l) or 0) for l in st.loop_labels]
    inner = loops[-2:]                        # fused into the launch (batch, batch2)
    outer = loops[:-2]
    while len(inner) < 2:
        inner.append((1, 0, 0, 0))
    (b1, apt, bpt, cpt), (b2, apt2, bpt2, cpt2) = inner
    for combo in itertools.product(*(range(e) for e, *_ in outer)):
        ox = sum(i * sx for i, (_, sx, _, _) in zip(combo, outer))
        oy = sum(i * sy for i, (_, _, sy, _) in zip(combo, outer))
        oc = sum(i * sc for i, (_, _, _, sc) in zip(combo, outer))
        core_call(m, 1, kk, alpha, bx.data, ox, ars, acs, apt, by.data, oy, brs, 1, bpt, beta,
                  c.data, oc, crs, 1, cpt, batch=b1, apt2=apt2, bpt2=bpt2, cpt2=cpt2,
                  batch2=b2)
        if counters is not None:
            counters.kernel_calls["gemv"] = counters.kernel_calls.get("gemv", 0) + 1


def _execute_conventional(plan, a, b, alpha, beta, c, counters):
    """Device execution of a conventional plan (reference planner.py:620-713):
    permute A / B / C into GEMM form with the library's permute kernel, one
    GEMM (level-2/1 families are the same GEMM with an extent of 1), permute
    the result back into C."""
    from .kernels import gemm
    info = plan.conventional
    spec = plan.spec

    def note_copy(n_elements):
        if counters is not None:
            counters.transpositions += 1
            counters.bytes_copied += n_elements * c.data.element_size()

    ta = a
    if info.permute_a is not None:
        ta = permute_copy(a, info.permute_a)
        note_copy(ta.layout.size)
    tb = b
    if info.permute_b is not None:
        tb = permute_copy(b, info.permute_b)
        note_copy(tb.layout.size)
    ext = {}
    for labels, lay in ((spec.labels_a, plan.layout_a), (spec.labels_b, plan.layout_b)):
        ext.update(dict(zip(labels, lay.dims)))
    mi = prod(ext[l] for l in info.free_a) if info.free_a else 1
    nj = prod(ext[l] for l in info.free_b) if info.free_b else 1
    kk = prod(ext[l] for l in info.contracted) if info.contracted else 1
    target_c = info.free_a + info.free_b
    if info.c_matches:
        cbuf = c
    else:
        cbuf = DenseTensor.zeros(Layout.packed([ext[l] for l in target_c] or [1]),
                                 dtype=c.dtype, device=c.device)
        if beta != 0.0 or info.policy == "naive":
            perm_in = tuple(spec.labels_c.index(l) for l in target_c)
            permute_into(c, perm_in, cbuf)
            note_copy(cbuf.layout.size)
    lda = kk if info.op_a is Op.Transpose else mi
    ldb = nj if info.op_b is Op.Transpose else kk
    gemm(info.op_a, info.op_b, mi, nj, kk, alpha, ta.data, lda, tb.data, ldb, beta,
         cbuf.data, mi)
    if counters is not None:
        fam = info.family.lower()
        counters.kernel_calls[fam] = counters.kernel_calls.get(fam, 0) + 1
    if not info.c_matches:
        perm_out = tuple(target_c.index(l) for l in spec.labels_c)
        permute_into(cbuf, perm_out, c)
        note_copy(c.layout.size)


def _storage_overlap(x, y) -> bool:
    """Whether the memory spans of two tensors intersect (for strided views the
    span from the lowest to the highest addressed element)."""
    if x.device != y.device:
        return False

    def span(t):
        lo = t.data_ptr()
        if t.numel() == 0:
            return lo, lo
        top = sum((d - 1) * s for d, s in zip(t.shape, t.stride()) if d > 0)
        return lo, lo + (top + 1) * t.element_size()
    xs, xe = span(x)
    ys, ye = span(y)
    return xs < ye and ys < xe


def _check_tensor(planned: Layout, t: DenseTensor, name: str):
    if t.layout != planned:
        raise PlanConsistencyError(
            f"layout of {name} drifted from the planned layout: {t.layout} != {planned}")


def execute_plan(plan: EvaluationPlan, a: DenseTensor, b: DenseTensor,
                 alpha: float, beta: float, c: DenseTensor,
                 threads: int = 1, counters=None) -> None:
    """Run a plan on device tensors, mutating C in place (one kernel launch
    per plan for every case with at most one loop mode)."""
    _check_tensor(plan.layout_a, a, "A")
    _check_tensor(plan.layout_b, b, "B")
    _check_tensor(plan.layout_c, c, "C")
    if _storage_overlap(c.data, a.data) or _storage_overlap(c.data, b.data):
        raise PlanError("C must not alias A or B")
    if plan.strategy == "conventional":
        _execute_conventional(plan, a, b, alpha, beta, c, counters)
        return
    if plan.strategy == "batched-gemv":
        _execute_gemv(plan, a, b, alpha, beta, c, counters)
        return
    if plan.strategy not in ("flattened-gemm", "strided-batched", "nested-batched",
                             "extended-batched"):
        raise PlanError(f"strategy {plan.strategy!r} is not executed by this backend")
    L = lower_plan(plan)
    x, y = (a.data, b.data) if L.first == "A" else (b.data, a.data)
    ars, acs, apt, apt2, brs, bcs, bpt, bpt2, crs, ccs, cpt, cpt2 = L.strides
    for ox, oy, oc in L.outer:
        core_call(L.m, L.n, L.k, alpha, x, ox, ars, acs, apt, y, oy, brs, bcs, bpt, beta,
                  c.data, oc, crs, ccs, cpt, batch=L.batch, apt2=apt2, bpt2=bpt2, cpt2=cpt2,
                  batch2=L.batch2, extended=L.extended)
        if counters is not None:
            counters.kernel_calls[L.kind] = counters.kernel_calls.get(L.kind, 0) + 1


def execute_plans(calls) -> None:
    """Run several INDEPENDENT planned contractions as one grouped call of the
    library (``sbt_batched_core_group_*``): the ones the CTA-pair tensor-core
    kernel takes share one persistent launch per kernel configuration, so a
    batch of contractions pays one pipeline fill / drain / tile tail instead of
    one per contraction.  ``calls`` is a sequence of
    (plan, a, b, alpha, beta, c) with the arguments of execute_plan.  No call's
    C may overlap another call's A, B or C (ValueError otherwise).  Single-mode
    plans only; results equal running execute_plan on each call."""
    import ctypes

    import torch

    from . import _lib
    from . import kernels as _k
    calls = list(calls)
    if not calls:
        return
    descs = []
    dtype = None
    device = None
    spans = []
    for plan, a, b, alpha, beta, c in calls:
        _check_tensor(plan.layout_a, a, "A")
        _check_tensor(plan.layout_b, b, "B")
        _check_tensor(plan.layout_c, c, "C")
        if _storage_overlap(c.data, a.data) or _storage_overlap(c.data, b.data):
            raise PlanError("C must not alias A or B")
        if plan.strategy not in ("flattened-gemm", "strided-batched", "nested-batched",
                                 "extended-batched"):
            raise PlanError(f"strategy {plan.strategy!r} cannot be grouped")
        if dtype is None:
            dtype, device = c.data.dtype, c.data.device
        if a.data.dtype != dtype or b.data.dtype != dtype or c.data.dtype != dtype:
            raise ValueError("grouped calls must share one dtype")
        if c.data.device != device or a.data.device != device or b.data.device != device:
            raise ValueError("grouped calls must share one device")
        L = lower_plan(plan)
        x, y = (a.data, b.data) if L.first == "A" else (b.data, a.data)
        ars, acs, apt, apt2, brs, bcs, bpt, bpt2, crs, ccs, cpt, cpt2 = L.strides
        for ox, oy, oc in L.outer:
            if L.batch == 0 or L.batch2 == 0:
                continue
            _k.validate_call(L.m, L.n, L.k, x, ox, ars, acs, apt, y, oy, brs, bcs, bpt,
                             c.data, oc, crs, ccs, cpt, L.batch, apt2, bpt2, cpt2, L.batch2)
            descs.append(_lib.GemmDesc(L.m, L.n, L.k, float(alpha), float(beta),
                                       x.data_ptr(), ox, ars, acs, apt, apt2,
                                       y.data_ptr(), oy, brs, bcs, bpt, bpt2,
                                       c.data.data_ptr(), oc, crs, ccs, cpt, cpt2,
                                       L.batch, L.batch2))
        spans.append((c.data, a.data, b.data))
    for i, (ci, _, _) in enumerate(spans):
        for j, (cj, aj, bj) in enumerate(spans):
            if i != j and (_storage_overlap(ci, cj) or _storage_overlap(ci, aj) or
                           _storage_overlap(ci, bj)):
                raise ValueError(f"grouped calls {i} and {j} are not independent "
                                 "(a C overlaps another call's operands)")
    if not descs:
        return
    arr = (_lib.GemmDesc * len(descs))(*descs)
    lib = _lib.load()
    fn = lib.sbt_batched_core_group_f64 if dtype == torch.float64 else \
        lib.sbt_batched_core_group_f32
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream(device).cuda_stream
        _lib.check(fn(len(descs), ctypes.cast(arr, ctypes.POINTER(_lib.GemmDesc)), stream),
                   "grouped strided batched GEMM")


# ---------------------------------------------------------------------------
# reporting


def _render_tensor(name, modes, batch_label=None):
    body = []
    for md in modes:
        text = md.label if len(md.label) == 1 else f"({md.label})"
        body.append(f"[{text}]" if md.label == batch_label else text)
    return f"{name}[{''.join(body)}]"


def render_plan(plan: EvaluationPlan) -> str:
    """Paper-style notation, one step per line (reference planner.py:730-781)."""
    gemm, batch = _gemm_and_batch(plan)
    blabel = batch.batch_label if batch else None
    lines, indent = [], ""
    for step in plan.steps:
        if isinstance(step, LoopStep):
            lines.append(f"{indent}for {step.label} in [0,{step.extent}):")
            indent += "  "
    second = "B" if gemm.first == "A" else "A"
    tf = "^T" if gemm.op_first in (Op.Transpose, Op.ExtendedTranspose) else ""
    ts = "^T" if gemm.op_second is Op.Transpose else ""
    lines.append(f"{indent}{_render_tensor('C', plan.eff['C'], blabel)} = "
                 f"{_render_tensor(gemm.first, plan.eff[gemm.first], blabel)}{tf} "
                 f"{_render_tensor(second, plan.eff[second], blabel)}{ts}")
    return "\n".join(lines)


def resolved_kernel_args(plan: EvaluationPlan, alpha=1.0, beta=0.0):
    """The reference's KernelArgs for the plan's (batched) GEMM step
    (planner.py:784-830): ld/lo in the op-flag convention of kernels.py."""
    last = plan.steps[-1] if plan.steps else None
    if not isinstance(last, (GemmStep, BatchedStep)):
        return None
    gemm, batch = _gemm_and_batch(plan)
    eff = {t: _ModeList(plan.eff[t]) for t in "ABC"}
    X, Y = (eff["A"], eff["B"]) if gemm.first == "A" else (eff["B"], eff["A"])
    C = eff["C"]
    ext = {md.label: md.extent for md in (*eff["A"], *eff["B"], *C)}
    m = ext[gemm.m_label] if gemm.m_label else 1
    n = ext[gemm.n_label] if gemm.n_label else 1
    k = ext[gemm.k_label]
    two = [md for md in X if md.label in (gemm.m_label, gemm.k_label)]
    if gemm.op_first is Op.Normal:
        lda = X.stride(gemm.k_label)
    elif gemm.op_first is Op.Transpose:
        lda = X.stride(gemm.m_label)
    else:
        lda = two[0].stride
    if gemm.op_second is Op.Normal:
        ldb = Y.stride(gemm.n_label) if gemm.n_label else k
    else:
        ldb = Y.stride(gemm.k_label)
    ldc = (C.stride(gemm.n_label) if gemm.n_label else max(m, 1)) or max(m, 1)
    loa = lob = loc = count = 0
    if batch is not None:
        count = batch.extent
        loc = C.stride(batch.batch_label)
        lob = Y.stride(batch.batch_label) or 0
        loa = two[1].stride if batch.extended else (X.stride(batch.batch_label) or 0)
    return KernelArgs(opa=gemm.op_first, opb=gemm.op_second, m=m, n=n, k=k,
                      alpha=alpha, beta=beta, lda=lda or max(m, 1), loa=loa,
                      ldb=ldb or k, lob=lob, ldc=ldc, loc=loc, batch_count=count)
