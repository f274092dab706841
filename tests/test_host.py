"""Host-side logic (no GPU): dispatcher parity with the reference's own plans,
notation and layout semantics, error behaviour, and the C-ABI library's
exported symbols."""
import re
from math import factorial
from pathlib import Path

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1606_05696_b200 as sbt
from paper_1606_05696_b200 import _lib, kernels
from paper_1606_05696_b200.kernels import Op
from paper_1606_05696_b200.layout import Layout
from paper_1606_05696_b200.notation import ContractionSpec, parse_contraction
from paper_1606_05696_b200.planner import (BatchedStep, LoopStep, PlanError,
                                           UnsupportedContractionError, enumerate_cases,
                                           find_case, lower_plan, plan_single_mode,
                                           render_plan, resolved_kernel_args)
from oracle import plan as oplan

ROOT = Path(__file__).resolve().parent.parent
EXCEPTIONAL = {"3.4", "3.6", "4.4", "4.6", "5.4", "5.6", "6.4", "6.6"}
SINGLE = {"1.1", "1.5", "2.1", "2.5", "5.1", "5.5", "6.1", "6.5"}


def _packed(spec, ext):
    return (Layout.packed([ext[l] for l in spec.labels_a]),
            Layout.packed([ext[l] for l in spec.labels_b]),
            Layout.packed([ext[l] for l in spec.labels_c] or [1]))


def _ka_dict(ka):
    return {"opa": ka.opa.value, "opb": ka.opb.value, "m": ka.m, "n": ka.n, "k": ka.k,
            "lda": ka.lda, "loa": ka.loa, "ldb": ka.ldb, "lob": ka.lob, "ldc": ka.ldc,
            "loc": ka.loc, "batch_count": ka.batch_count}


# ---------------------------------------------------------------- dispatcher


def test_partition_36_cases():
    cases = enumerate_cases(2, 3)
    assert len(cases) == 36 and len({c.case_id for c in cases}) == 36
    by = {}
    for c in cases:
        by.setdefault(c.classification, set()).add(c.case_id)
    assert by["single-gemm"] == SINGLE
    assert by["exceptional"] == EXCEPTIONAL
    assert len(by["strided-batched"]) == 20


def test_count_law():
    for a in (1, 2, 3):
        for b in (1, 2, 3):
            assert len(enumerate_cases(a, b)) == factorial(a + b - 2) * a * b


def test_catalogue_matches_reference(golden_plans):
    want = {(tuple(r["orders"]), r["case_id"]): r for r in golden_plans["cases"]}
    for oa in (1, 2, 3):
        for ob in (1, 2, 3):
            for case in enumerate_cases(oa, ob):
                ref = want[((oa, ob), case.case_id)]
                assert "".join(case.labels_a) == ref["labels_a"]
                assert "".join(case.labels_b) == ref["labels_b"]
                assert "".join(case.labels_c) == ref["labels_c"]
                assert case.classification == ref["classification"]


def test_plans_match_reference_exactly(golden_plans):
    """Strategy, steps, effective modes, render text and KernelArgs for every
    case of every (a, b) order pair at 5 extent sets."""
    for rec in golden_plans["cases"]:
        spec = ContractionSpec(tuple(rec["labels_a"]), tuple(rec["labels_b"]),
                               tuple(rec["labels_c"]))
        for p in rec["plans"]:
            plan = plan_single_mode(spec, *_packed(spec, p["ext"]))
            where = (rec["orders"], rec["case_id"], p["ext"])
            assert plan.strategy == p["strategy"], where
            assert {t: [[m.label, m.extent, m.stride] for m in plan.eff[t]] for t in "ABC"} \
                == p["eff"], where
            assert render_plan(plan) == p["render"], where
            assert _ka_dict(resolved_kernel_args(plan)) == p["kernel_args"], where


def test_extra_plans_match_reference(golden_plans):
    for ex in golden_plans["extra"]:
        spec = ContractionSpec(tuple(ex["a"]), tuple(ex["b"]), tuple(ex["c"]))
        lays = [Layout(tuple(d), tuple(s)) for d, s in ex["layouts"]]
        plan = plan_single_mode(spec, *lays)
        assert plan.strategy == ex["strategy"], ex["name"]
        assert render_plan(plan) == ex["render"], ex["name"]
        assert _ka_dict(resolved_kernel_args(plan)) == ex["kernel_args"], ex["name"]


def test_lowering_matches_oracle_core_calls(golden_plans):
    """The device launch (true element strides, fused loop) addresses exactly
    the elements the reference's core calls address."""
    for rec in golden_plans["cases"]:
        if rec["orders"] != [2, 3]:
            continue
        spec = ContractionSpec(tuple(rec["labels_a"]), tuple(rec["labels_b"]),
                               tuple(rec["labels_c"]))
        for p in rec["plans"]:
            la, lb, lc = _packed(spec, p["ext"])
            L = lower_plan(plan_single_mode(spec, la, lb, lc))
            low = oplan.lower(spec.labels_a, spec.labels_b, spec.labels_c, la.dims, la.strides,
                              lb.dims, lb.strides, lc.dims, lc.strides)
            assert L.first == low["first"]
            assert len(low["calls"]) == 1
            cl = low["calls"][0]
            ars, acs, apt, _, brs, bcs, bpt, _, crs, ccs, cpt, _ = L.strides
            assert (L.m, L.n, L.k) == (cl["m"], cl["n"], cl["k"])
            assert L.batch == cl["batch"]
            # rows/cols with extent 1 may carry any stride
            if L.m > 1:
                assert ars == cl["ars"] and crs == cl["crs"]
            if L.n > 1:
                assert bcs == cl["bcs"] and ccs == cl["ccs"]
            assert acs == cl["acs"] or L.k == 1
            assert brs == cl["brs"] or L.k == 1
            if L.batch > 1:
                assert (apt, bpt, cpt) == (cl["apt"], cl["bpt"], cl["cpt"])


def test_nested_plan_fuses_loop_into_one_launch():
    spec = ContractionSpec(tuple("mkp"), tuple("nkq"), tuple("mnpq"))
    for p, q in ((4, 7), (7, 4)):
        ext = dict(m=5, n=6, k=3, p=p, q=q)
        plan = plan_single_mode(spec, *_packed(spec, ext))
        assert plan.strategy == "nested-batched"
        step = plan.steps[-1]
        assert isinstance(step, BatchedStep) and step.batch_label == ("p" if p > q else "q")
        assert sum(isinstance(s, LoopStep) for s in plan.steps) == 1
        L = lower_plan(plan)
        assert L.batch == max(p, q) and L.batch2 == min(p, q) and len(L.outer) == 1


def test_case_1_1_flattens():
    spec = parse_contraction("C[mnp] = A[mk] * B[knp]")
    plan = plan_single_mode(spec, *_packed(spec, dict(m=4, n=5, p=6, k=3)))
    assert plan.strategy == "flattened-gemm"
    ka = resolved_kernel_args(plan)
    assert (ka.m, ka.n, ka.k) == (4, 30, 3)
    assert "C[m(np)] = A[mk] B[k(np)]" in render_plan(plan)


def test_stride_gap_blocks_flattening():
    spec = parse_contraction("C[mnp] = A[mk] * B[knp]")
    plan = plan_single_mode(spec, Layout.packed([4, 3]), Layout((3, 5, 6), (1, 3, 16)),
                            Layout.packed([4, 5, 6]))
    assert plan.strategy == "strided-batched"


def test_plan_errors():
    spec = ContractionSpec(("m", "k", "l"), ("k", "l", "n"), ("m", "n"))
    with pytest.raises(UnsupportedContractionError):
        plan_single_mode(spec, Layout.packed([2, 3, 4]), Layout.packed([3, 4, 5]),
                         Layout.packed([2, 5]))
    spec = parse_contraction("C[mn] = A[mk] * B[kn]")
    with pytest.raises(PlanError):
        plan_single_mode(spec, Layout.packed([4, 3]), Layout.packed([2, 5]),
                         Layout.packed([4, 5]))
    with pytest.raises(PlanError):
        find_case(2, 3, "9.9")


def test_extent_one_modes_squeezed():
    spec = parse_contraction("C[mnp] = A[mk] * B[knp]")
    plan = plan_single_mode(spec, Layout.packed([4, 3]), Layout.packed([3, 1, 6]),
                            Layout.packed([4, 1, 6]))
    assert "n" not in {m.label for m in plan.eff["C"]}


# ---------------------------------------------------------------- notation / layout


def test_notation_grammar():
    spec = parse_contraction("C[mnp] = 2.5 A[mk] * B[knp] + 0.5 C[mnp]")
    assert spec.alpha == 2.5 and spec.beta == 0.5
    assert spec.contracted == ("k",)
    for bad in ("C[mn] = A[mk] * B[kn] + 1 C[nm]", "C[mn] = A[mmk] * B[kn]",
                "C[m] = A[mk] * B[kn]", "C[mn] = A[mk] + B[kn]"):
        with pytest.raises(ValueError):
            parse_contraction(bad)
    assert sbt.format_contraction(spec) == "C[mnp] = 2.5 A[mk] * B[knp] + 0.5 C[mnp]"
    cls = sbt.classify_indices(spec)
    assert sbt.kernel_family(cls) == "GEMM"


def test_layout_rules():
    assert Layout.packed([4, 5, 6]).strides == (1, 4, 20)
    for dims, strides in (((0, 3), (1, 1)), ((2, 3), (2, 2)), ((2,), (1, 1)), ((3, 3), (1, 1))):
        with pytest.raises(ValueError):
            Layout(dims, strides)
    lay = Layout.packed([4, 5, 6])
    assert sbt.can_flatten(lay, 0, 1) and not sbt.can_flatten(lay, 0, 2)
    assert sbt.flatten(lay, 0, 1) == Layout((20, 6), (1, 20))
    with pytest.raises(sbt.IllegalFlattenError):
        sbt.flatten(Layout((4, 5), (1, 8)), 0, 1)
    assert sbt.linear_offset(Layout.packed([3, 4]), (2, 3)) == 11


@settings(max_examples=50, deadline=None)
@given(dims=st.lists(st.integers(2, 4), min_size=2, max_size=4), data=st.data())
def test_flatten_preserves_offsets(dims, data):
    lay = Layout.packed(dims)
    i = data.draw(st.integers(0, len(dims) - 2))
    merged = sbt.flatten(lay, i, i + 1)
    x = data.draw(st.integers(0, dims[i] - 1))
    y = data.draw(st.integers(0, dims[i + 1] - 1))
    idx = [0] * len(dims)
    idx[i], idx[i + 1] = x, y
    midx = list(idx)
    del midx[i + 1]
    midx[i] = x + y * dims[i]
    assert sbt.linear_offset(lay, idx) == sbt.linear_offset(merged, midx)


# ---------------------------------------------------------------- kernel API validation


def test_kernel_validation_errors():
    z = np.zeros(64)
    with pytest.raises(ValueError):
        kernels.gemm(Op.ExtendedNormal, Op.Normal, 2, 2, 2, 1.0, z, 2, z, 2, 0.0, z.copy(), 2)
    with pytest.raises(ValueError):
        kernels.gemm(Op.Normal, Op.Normal, 4, 2, 2, 1.0, z, 2, z, 2, 0.0, z.copy(), 4)
    with pytest.raises(ValueError):
        kernels.gemm("C", Op.Normal, 2, 2, 2, 1.0, z, 2, z, 2, 0.0, z.copy(), 2)
    with pytest.raises(ValueError):
        kernels.strided_batched_gemm(Op.Normal, Op.Normal, 4, 4, 2, 1.0, z, 4, 0, z, 2, 0,
                                     0.0, z.copy(), 4, 1, 3)
    with pytest.raises(ValueError):
        kernels.strided_batched_gemm_ex(Op.Normal, Op.Normal, 2, 2, 2, 1.0, z, 2, 4, z, 2, 4,
                                        0.0, z.copy(), 2, 4, 2)
    with pytest.raises(ValueError):
        kernels.strided_batched_gemm(Op.Normal, Op.Normal, 0, 2, 2, 1.0, z, 2, 4, z, 2, 4,
                                     0.0, z.copy(), 2, 4, 2)
    # batch 0 is a no-op before any buffer is touched
    c = np.full(8, 5.0)
    kernels.strided_batched_gemm(Op.Normal, Op.Normal, 2, 2, 2, 1.0, np.zeros(8), 2, 4,
                                 np.zeros(8), 2, 4, 0.0, c, 2, 4, 0)
    np.testing.assert_array_equal(c, np.full(8, 5.0))


def test_out_of_bounds_is_rejected_before_launch():
    a = np.zeros(10)
    with pytest.raises(ValueError, match="addresses element"):
        kernels.gemm(Op.Normal, Op.Normal, 4, 4, 4, 1.0, a, 4, a, 4, 0.0, np.zeros(16), 4)


# ---------------------------------------------------------------- C ABI


def _header_symbols():
    text = (ROOT / "include" / "sbt200.h").read_text()
    return sorted(set(re.findall(r"\b(sbt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.SIGNATURES)
    assert lib.sbt_version() >= 100


def test_library_rejects_bad_arguments_without_gpu():
    lib = _lib.load()
    # validation precedes any CUDA call: negative extent / stride, null pointers
    rc = lib.sbt_batched_core_f64(-1, 2, 2, 1.0, 0, 0, 1, 2, 0, 0, 0, 1, 2, 0, 0.0, 0, 0, 1, 2,
                                  0, 1, None)
    assert rc == _lib.SBT_EINVAL
    assert "extent" in lib.sbt_last_error().decode()
    rc = lib.sbt_gemm_core_f32(2, 2, 2, 1.0, None, 0, 1, 2, None, 0, 1, 2, 0.0, None, 0, 1, 2,
                               None)
    assert rc == _lib.SBT_EINVAL
    assert lib.sbt_set_kernel_override(7) == _lib.SBT_EINVAL
