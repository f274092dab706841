"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container only (the reference tree is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Everything is produced by calling the unmodified reference package
(`sbtensor`, /root/reference/pkg/src) through its public API:

* plans.json      -- plan_single_mode / resolved_kernel_args / render_plan for
                     every case of enumerate_cases(a, b), a, b in 1..3, at
                     canonical, square and randomly drawn extents
                     (planner.py:132-371, :784-830);
* contract.npz    -- execute_plan outputs for all 36 (2,3) cases at random
                     extents in [1, 8] with random alpha/beta and random C
                     (test_acceptance.py:63-81 protocol), plus nested 4th-order
                     and padded-stride examples;
* kernels.npz     -- strided_batched_gemm / strided_batched_gemm_ex / gemm
                     outputs on the reference's own test shapes
                     (test_kernels.py:12-135) and strided variants;
* hooi.npz        -- hooi() results (factors, core, fit history) on the
                     reference's Tucker test tensors (test_tucker.py:54-94,
                     test_acceptance.py:182-201);
* conventional.*  -- plan_conventional plans (steps, ops, transposition count)
                     and contract_conventional outputs + counters for all 36
                     (2,3) cases, both policies, beta = 0 and != 0
                     (planner.py:411-465, 620-713; reference.py:54-63).
                     ``--only conventional`` regenerates just these.

The fixtures are small (<1 MB) and committed; this script is committed next to
them so they can be regenerated.
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("SBT_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import sbtensor  # noqa: E402
from sbtensor import kernels  # noqa: E402
from sbtensor.kernels import Op  # noqa: E402
from sbtensor.layout import DenseTensor, Layout  # noqa: E402
from sbtensor.notation import ContractionSpec  # noqa: E402
from sbtensor.planner import (BatchedStep, FlattenStep, GemmStep, GemvBatchStep,  # noqa: E402
                              LoopStep, PermuteStep, enumerate_cases, execute_plan,
                              plan_batched_gemv, plan_conventional, plan_single_mode,
                              render_plan, resolved_kernel_args)
from sbtensor.reference import contract_conventional  # noqa: E402
from sbtensor.tucker import hooi, tucker_core, tucker_reconstruct  # noqa: E402

OUT = Path(__file__).resolve().parent


def _step_json(step):
    if isinstance(step, FlattenStep):
        return {"type": "flatten", "tensor": step.tensor, "labels": list(step.labels),
                "merged": step.merged}
    if isinstance(step, LoopStep):
        return {"type": "loop", "label": step.label, "extent": step.extent}
    if isinstance(step, GemmStep):
        return {"type": "gemm", "first": step.first, "op_first": step.op_first.value,
                "op_second": step.op_second.value, "m_label": step.m_label,
                "n_label": step.n_label, "k_label": step.k_label}
    if isinstance(step, BatchedStep):
        return {"type": "batched", "gemm": _step_json(step.gemm),
                "batch_label": step.batch_label, "extent": step.extent,
                "extended": step.extended}
    raise TypeError(step)


def _plan_json(plan):
    ka = resolved_kernel_args(plan)
    return {
        "strategy": plan.strategy,
        "steps": [_step_json(s) for s in plan.steps],
        "eff": {t: [[m.label, m.extent, m.stride] for m in plan.eff[t]] for t in "ABC"},
        "render": render_plan(plan),
        "kernel_args": None if ka is None else {
            "opa": ka.opa.value, "opb": ka.opb.value, "m": ka.m, "n": ka.n, "k": ka.k,
            "lda": ka.lda, "loa": ka.loa, "ldb": ka.ldb, "lob": ka.lob,
            "ldc": ka.ldc, "loc": ka.loc, "batch_count": ka.batch_count},
    }


def make_plans(rng):
    out = []
    for oa in (1, 2, 3):
        for ob in (1, 2, 3):
            for case in enumerate_cases(oa, ob):
                spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
                labels = sorted(set(spec.labels_a) | set(spec.labels_b))
                ext_sets = [
                    {l: 3 + i for i, l in enumerate(labels)},
                    {l: 256 for l in labels},
                ]
                for _ in range(3):
                    ext_sets.append({l: int(rng.integers(1, 7)) for l in labels})
                rec = {"orders": [oa, ob], "case_id": case.case_id,
                       "labels_a": "".join(case.labels_a), "labels_b": "".join(case.labels_b),
                       "labels_c": "".join(case.labels_c),
                       "classification": case.classification, "plans": []}
                for ext in ext_sets:
                    la = Layout.packed([ext[l] for l in spec.labels_a])
                    lb = Layout.packed([ext[l] for l in spec.labels_b])
                    lc = Layout.packed([ext[l] for l in spec.labels_c] or [1])
                    plan = plan_single_mode(spec, la, lb, lc)
                    rec["plans"].append({"ext": ext, **_plan_json(plan)})
                out.append(rec)
    # nested 4th-order spec and a padded-stride example (test_planner.py:48-56, :99-113)
    extra = []
    spec = ContractionSpec(tuple("mkp"), tuple("nkq"), tuple("mnpq"))
    for p, q in ((4, 7), (7, 4), (5, 5), (128, 128)):
        ext = dict(m=5, n=6, k=3, p=p, q=q) if p != 128 else dict(m=128, n=128, k=128, p=128, q=128)
        la = Layout.packed([ext[l] for l in spec.labels_a])
        lb = Layout.packed([ext[l] for l in spec.labels_b])
        lc = Layout.packed([ext[l] for l in spec.labels_c])
        extra.append({"name": f"nested_p{p}_q{q}", "a": "mkp", "b": "nkq", "c": "mnpq",
                      "layouts": [[la.dims, la.strides], [lb.dims, lb.strides], [lc.dims, lc.strides]],
                      **_plan_json(plan_single_mode(spec, la, lb, lc))})
    spec = ContractionSpec(tuple("mk"), tuple("knp"), tuple("mnp"))
    la, lb, lc = Layout.packed([4, 3]), Layout((3, 5, 6), (1, 3, 16)), Layout.packed([4, 5, 6])
    extra.append({"name": "padded_b", "a": "mk", "b": "knp", "c": "mnp",
                  "layouts": [[la.dims, la.strides], [lb.dims, lb.strides], [lc.dims, lc.strides]],
                  **_plan_json(plan_single_mode(spec, la, lb, lc))})
    return {"cases": out, "extra": extra}


def make_contract(rng):
    arrays = {}
    index = []
    for case in enumerate_cases(2, 3):
        spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
        for rep in range(3):
            ext = {l: int(rng.integers(1, 9)) for l in "mnpk"}
            alpha = float(rng.uniform(-2, 2))
            beta = float(rng.uniform(-2, 2)) if rep else 0.0
            la = Layout.packed([ext[l] for l in spec.labels_a])
            lb = Layout.packed([ext[l] for l in spec.labels_b])
            lc = Layout.packed([ext[l] for l in spec.labels_c])
            a = DenseTensor.from_array(rng.uniform(-1, 1, la.dims))
            b = DenseTensor.from_array(rng.uniform(-1, 1, lb.dims))
            c = DenseTensor.from_array(rng.uniform(-1, 1, lc.dims))
            key = f"{case.case_id}_{rep}"
            arrays[key + "_a"] = a.data.copy()
            arrays[key + "_b"] = b.data.copy()
            arrays[key + "_c0"] = c.data.copy()
            plan = plan_single_mode(spec, la, lb, lc)
            execute_plan(plan, a, b, alpha, beta, c)
            arrays[key + "_c"] = c.data.copy()
            index.append({"key": key, "case_id": case.case_id, "a": "".join(spec.labels_a),
                          "b": "".join(spec.labels_b), "c": "".join(spec.labels_c),
                          "ext": ext, "alpha": alpha, "beta": beta})
    # nested 4th-order: C[mnpq] = A[mkp] B[nkq]
    spec = ContractionSpec(tuple("mkp"), tuple("nkq"), tuple("mnpq"))
    for p, q in ((4, 7), (7, 4)):
        ext = dict(m=5, n=6, k=3, p=p, q=q)
        la = Layout.packed([ext[l] for l in spec.labels_a])
        lb = Layout.packed([ext[l] for l in spec.labels_b])
        lc = Layout.packed([ext[l] for l in spec.labels_c])
        a = DenseTensor.from_array(rng.uniform(-1, 1, la.dims))
        b = DenseTensor.from_array(rng.uniform(-1, 1, lb.dims))
        c = DenseTensor.zeros(lc)
        key = f"nested_{p}_{q}"
        arrays[key + "_a"] = a.data.copy()
        arrays[key + "_b"] = b.data.copy()
        arrays[key + "_c0"] = c.data.copy()
        execute_plan(plan_single_mode(spec, la, lb, lc), a, b, 1.0, 0.0, c)
        arrays[key + "_c"] = c.data.copy()
        index.append({"key": key, "case_id": "nested", "a": "mkp", "b": "nkq", "c": "mnpq",
                      "ext": ext, "alpha": 1.0, "beta": 0.0})
    return arrays, index


def _fvec(arr):
    return np.asfortranarray(arr).reshape(-1, order="F")


def make_kernels(rng):
    """Reference kernel outputs; each record stores the exact keyword arguments."""
    arrays = {}
    index = []

    def record(name, fn, kw, a, b, c0):
        c = c0.copy()
        getattr(kernels, fn)(a=a, b=b, c=c, **kw)
        arrays[name + "_a"], arrays[name + "_b"] = a.copy(), b.copy()
        arrays[name + "_c0"], arrays[name + "_c"] = c0.copy(), c
        index.append({"name": name, "fn": fn,
                      "kw": {k: (v.value if isinstance(v, Op) else v) for k, v in kw.items()}})

    def sb(opa, opb, m, n, k, alpha, lda, loa, ldb, lob, beta, ldc, loc, batch, **extra):
        return dict(opa=opa, opb=opb, m=m, n=n, k=k, alpha=alpha, lda=lda, loa=loa,
                    ldb=ldb, lob=lob, beta=beta, ldc=ldc, loc=loc, batch_count=batch, **extra)

    # gemm, all op combos, beta != 0 (test_kernels.py:12-25)
    for opa in (Op.Normal, Op.Transpose):
        for opb in (Op.Normal, Op.Transpose):
            m, n, k = 4, 5, 3
            A = rng.standard_normal((m, k) if opa is Op.Normal else (k, m))
            B = rng.standard_normal((k, n) if opb is Op.Normal else (n, k))
            C = rng.standard_normal((m, n))
            record(f"gemm_{opa.value}{opb.value}", "gemm",
                   dict(opa=opa, opb=opb, m=m, n=n, k=k, alpha=1.5, lda=A.shape[0],
                        ldb=B.shape[0], beta=0.5, ldc=m),
                   _fvec(A), _fvec(B), _fvec(C))
    # gemm with padded leading dims and offsets
    m, n, k = 7, 6, 5
    record("gemm_padded", "gemm",
           dict(opa=Op.Normal, opb=Op.Normal, m=m, n=n, k=k, alpha=-0.75, lda=9, ldb=8,
                beta=1.25, ldc=11, offa=3, offb=2, offc=4),
           rng.standard_normal(9 * k + 3), rng.standard_normal(8 * n + 2),
           rng.standard_normal(11 * n + 4))
    # strided batched, packed (test_kernels.py:70-81)
    m, n, k, P = 4, 5, 3, 6
    A = rng.standard_normal((m, k, P))
    B = rng.standard_normal((k, n, P))
    record("sbgemm_packed", "strided_batched_gemm",
           sb(Op.Normal, Op.Normal, m, n, k, 1.0, m, m * k, k, k * n, 0.0, m, m * n, P),
           _fvec(A), _fvec(B), np.zeros(m * n * P))
    # lob = 0 broadcast (test_kernels.py:84-96)
    m, n, k, P = 3, 4, 2, 5
    A = rng.standard_normal((m, k, P))
    B = rng.standard_normal((k, n))
    record("sbgemm_broadcast", "strided_batched_gemm",
           sb(Op.Normal, Op.Normal, m, n, k, 1.0, m, m * k, k, 0, 0.0, m, m * n, P),
           _fvec(A), _fvec(B), np.zeros(m * n * P))
    # transposed ops, interleaved C (C[m[n]p] style), beta != 0
    m, n, k, P = 6, 7, 4, 9
    record("sbgemm_TT_interleaved", "strided_batched_gemm",
           sb(Op.Transpose, Op.Transpose, m, n, k, 0.8, k, k * m, n, n * k, -0.3, m * P, m, P),
           rng.standard_normal(k * m * P), rng.standard_normal(n * k * P),
           rng.standard_normal(m * P * n))
    # threads > 1 must equal threads = 1 (test_kernels.py:138-150)
    m, n, k, P = 6, 7, 4, 9
    A = rng.standard_normal((m, k, P))
    B = rng.standard_normal((k, n, P))
    record("sbgemm_threads3", "strided_batched_gemm",
           sb(Op.Normal, Op.Normal, m, n, k, 1.0, m, m * k, k, k * n, 0.0, m, m * n, P,
              threads=3),
           _fvec(A), _fvec(B), np.zeros(m * n * P))
    # extended ops on A (test_kernels.py:114-127) and on B
    for exop in (Op.ExtendedNormal, Op.ExtendedTranspose):
        m, n, k, P = 3, 4, 2, 5
        lda, loa = (P, P * m) if exop is Op.ExtendedNormal else (P, P * k)
        record(f"ex_A_{exop.value}", "strided_batched_gemm_ex",
               sb(exop, Op.Normal, m, n, k, 1.0, lda, loa, k, 0, 0.0, m, m * n, P),
               rng.standard_normal(P * m * k + 7), rng.standard_normal(max(k, n) ** 2 + 40),
               np.zeros(m * n * P))
        # B extended: B stored (p, k, n) [EN] or (p, n, k) [ET]; beta != 0
        ldb, lob = (P, P * k) if exop is Op.ExtendedNormal else (P, P * n)
        record(f"ex_B_{exop.value}", "strided_batched_gemm_ex",
               sb(Op.Normal, exop, m, n, k, 1.25, m, m * k, ldb, lob, 0.5, m, m * n, P),
               rng.standard_normal(m * k * P), rng.standard_normal(P * k * n + 5),
               rng.standard_normal(m * n * P))
    return arrays, index


def make_hooi(rng):
    arrays = {}
    index = []

    def exact_rank(dims, ranks):
        core = rng.standard_normal(ranks)
        factors = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
        return np.einsum("abc,ia,jb,kc->ijk", core, *factors)

    cases = [
        ("exact_12_11_10", exact_rank((12, 11, 10), (3, 2, 4)), (3, 2, 4), 20),
        ("random_10", rng.standard_normal((10, 10, 10)), (3, 3, 3), 10),
        ("full_5_6_4", rng.standard_normal((5, 6, 4)), (5, 6, 4), 5),
        ("exact_30", exact_rank((30, 30, 30), (4, 4, 4)), (4, 4, 4), 20),
        ("noisy_16", exact_rank((16, 16, 16), (4, 4, 4)) + 1e-3 * rng.standard_normal((16, 16, 16)),
         (4, 4, 4), 8),
    ]
    for name, arr, ranks, iters in cases:
        t = DenseTensor.from_array(arr)
        model = hooi(t, ranks, max_iters=iters)
        arrays[name + "_t"] = t.data.copy()
        for r, u in enumerate(model.factors):
            arrays[f"{name}_u{r}"] = u.copy()
        arrays[name + "_core"] = model.core.data.copy()
        arrays[name + "_rec"] = tucker_reconstruct(model).data.copy()
        arrays[name + "_core_of_t"] = tucker_core(t, model.factors).data.copy()
        index.append({"name": name, "dims": list(arr.shape), "ranks": list(ranks),
                      "max_iters": iters, "iterations": model.iterations,
                      "fit_history": model.fit_history})
    return arrays, index


def make_conventional(rng):
    arrays = {}
    index = []
    for case in enumerate_cases(2, 3):
        for policy in ("opt", "naive"):
            for rep in range(2):
                ext = {l: int(rng.integers(2, 8)) for l in "mnpk"}
                alpha = float(rng.uniform(-2, 2))
                beta = float(rng.uniform(-2, 2)) if rep else 0.0
                spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c,
                                       alpha=alpha, beta=beta)
                la = Layout.packed([ext[l] for l in spec.labels_a])
                lb = Layout.packed([ext[l] for l in spec.labels_b])
                lc = Layout.packed([ext[l] for l in spec.labels_c])
                plan = plan_conventional(spec, la, lb, lc, policy=policy)
                info = plan.conventional
                a = DenseTensor.from_array(rng.uniform(-1, 1, la.dims))
                b = DenseTensor.from_array(rng.uniform(-1, 1, lb.dims))
                c = DenseTensor.from_array(rng.uniform(-1, 1, lc.dims))
                key = f"{case.case_id}_{policy}_{rep}"
                arrays[key + "_a"] = a.data.copy()
                arrays[key + "_b"] = b.data.copy()
                arrays[key + "_c0"] = c.data.copy()
                counters = contract_conventional(spec, a, b, alpha, beta, c, policy=policy)
                arrays[key + "_c"] = c.data.copy()
                index.append({
                    "key": key, "case_id": case.case_id, "policy": policy,
                    "a": "".join(spec.labels_a), "b": "".join(spec.labels_b),
                    "c": "".join(spec.labels_c), "ext": ext, "alpha": alpha, "beta": beta,
                    "steps": [[st.tensor, list(st.perm)] for st in plan.steps
                              if isinstance(st, PermuteStep)],
                    "predicted_transpositions": plan.predicted_transpositions,
                    "op_a": info.op_a.value, "op_b": info.op_b.value,
                    "permute_a": None if info.permute_a is None else list(info.permute_a),
                    "permute_b": None if info.permute_b is None else list(info.permute_b),
                    "c_matches": info.c_matches, "family": info.family,
                    "transpositions": counters.transpositions,
                    "kernel_calls": counters.kernel_calls})
    # batched-GEMV strategy (planner.py:374-404, 584-617)
    for case in enumerate_cases(2, 3):
        for rep in range(2):
            ext = {l: int(rng.integers(2, 8)) for l in "mnpk"}
            alpha = float(rng.uniform(-2, 2))
            beta = float(rng.uniform(-2, 2)) if rep else 0.0
            spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
            la = Layout.packed([ext[l] for l in spec.labels_a])
            lb = Layout.packed([ext[l] for l in spec.labels_b])
            lc = Layout.packed([ext[l] for l in spec.labels_c])
            plan = plan_batched_gemv(spec, la, lb, lc)
            step = plan.steps[-1]
            assert isinstance(step, GemvBatchStep)
            a = DenseTensor.from_array(rng.uniform(-1, 1, la.dims))
            b = DenseTensor.from_array(rng.uniform(-1, 1, lb.dims))
            c = DenseTensor.from_array(rng.uniform(-1, 1, lc.dims))
            key = f"gemv_{case.case_id}_{rep}"
            arrays[key + "_a"] = a.data.copy()
            arrays[key + "_b"] = b.data.copy()
            arrays[key + "_c0"] = c.data.copy()
            execute_plan(plan, a, b, alpha, beta, c)
            arrays[key + "_c"] = c.data.copy()
            index.append({
                "key": key, "case_id": case.case_id, "policy": "batched-gemv",
                "a": "".join(spec.labels_a), "b": "".join(spec.labels_b),
                "c": "".join(spec.labels_c), "ext": ext, "alpha": alpha, "beta": beta,
                "flatten": [[st.tensor, list(st.labels), st.merged] for st in plan.steps
                            if isinstance(st, FlattenStep)],
                "gemv": {"loop_labels": list(step.loop_labels), "matrix": step.matrix,
                         "op": step.op.value, "v_label": step.v_label,
                         "k_label": step.k_label}})
    return arrays, index


def main():
    rng = np.random.default_rng(20260824)
    if "--only" in sys.argv and sys.argv[sys.argv.index("--only") + 1] == "conventional":
        meta = {"reference": REF, "sbtensor_version": sbtensor.__version__,
                "backend": sbtensor.active_backend(), "numpy": np.__version__}
        arrays, index = make_conventional(np.random.default_rng(1606))
        np.savez_compressed(OUT / "conventional.npz", **arrays)
        (OUT / "conventional.json").write_text(
            json.dumps({"meta": meta, "records": index}, indent=0))
        print("wrote conventional fixtures to", OUT)
        return
    meta = {"reference": REF, "sbtensor_version": sbtensor.__version__,
            "backend": sbtensor.active_backend(), "numpy": np.__version__}
    plans = make_plans(rng)
    (OUT / "plans.json").write_text(json.dumps({"meta": meta, **plans}, separators=(",", ":")))
    arrays, index = make_contract(rng)
    np.savez_compressed(OUT / "contract.npz", **arrays)
    (OUT / "contract.json").write_text(json.dumps({"meta": meta, "records": index}, indent=0))
    arrays, index = make_kernels(rng)
    np.savez_compressed(OUT / "kernels.npz", **arrays)
    (OUT / "kernels.json").write_text(json.dumps({"meta": meta, "records": index}, indent=0))
    arrays, index = make_hooi(rng)
    np.savez_compressed(OUT / "hooi.npz", **arrays)
    (OUT / "hooi.json").write_text(json.dumps({"meta": meta, "records": index}, indent=0))
    print("wrote golden fixtures to", OUT)


if __name__ == "__main__":
    main()
