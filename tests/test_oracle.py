"""Pin the CPU oracle against the golden fixtures produced by the real
reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle import api, naive, plan as oplan, tucker as otucker
from oracle.cores import batched_core, gemm_core, gemm_core_loops


def _lower_packed(rec, ext):
    la, lb, lc = rec["labels_a"], rec["labels_b"], rec["labels_c"]
    da = [ext[l] for l in la]
    db = [ext[l] for l in lb]
    dc = [ext[l] for l in lc] or [1]
    return oplan.lower(la, lb, lc, da, oplan.packed_strides(da), db, oplan.packed_strides(db),
                       dc, oplan.packed_strides(dc))


def test_oracle_planner_matches_reference_plans(golden_plans):
    n = 0
    for rec in golden_plans["cases"]:
        for p in rec["plans"]:
            low = _lower_packed(rec, p["ext"])
            assert low["strategy"] == p["strategy"], (rec["case_id"], p["ext"])
            assert low["args"] == {k: p["kernel_args"][k] for k in low["args"]}, \
                (rec["orders"], rec["case_id"], p["ext"])
            n += 1
    assert n == 5 * sum(1 for _ in golden_plans["cases"])


def test_oracle_planner_nested_and_padded(golden_plans):
    for ex in golden_plans["extra"]:
        (da, sa), (db, sb), (dc, sc) = ex["layouts"]
        low = oplan.lower(ex["a"], ex["b"], ex["c"], da, sa, db, sb, dc, sc)
        assert low["strategy"] == ex["strategy"], ex["name"]
        assert low["args"] == {k: ex["kernel_args"][k] for k in low["args"]}, ex["name"]


def test_oracle_contract_matches_reference_outputs(golden_contract):
    index, arr = golden_contract
    for rec in index["records"]:
        key = rec["key"]
        c = arr[key + "_c0"].copy()
        oplan.contract(rec["a"], rec["b"], rec["c"], rec["ext"], arr[key + "_a"],
                       arr[key + "_b"], rec["alpha"], rec["beta"], c)
        assert naive.max_rel_err(c, arr[key + "_c"]) <= 1e-13, key


def test_naive_oracle_matches_reference_outputs(golden_contract):
    index, arr = golden_contract
    for rec in index["records"][::7]:
        key = rec["key"]
        ext = rec["ext"]
        c = arr[key + "_c0"].copy()
        s = {t: oplan.packed_strides([ext[l] for l in rec[t]]) for t in "abc"}
        naive.contract_naive(rec["a"], rec["b"], rec["c"], ext, s["a"], s["b"], s["c"],
                             arr[key + "_a"], arr[key + "_b"], rec["alpha"], rec["beta"], c)
        assert naive.max_rel_err(c, arr[key + "_c"]) <= 1e-13, key


def test_oracle_kernel_calls_match_reference(golden_kernels):
    index, arr = golden_kernels
    for rec in index["records"]:
        name = rec["name"]
        c = arr[name + "_c0"].copy()
        api.run_call(rec["fn"], rec["kw"], arr[name + "_a"], arr[name + "_b"], c)
        np.testing.assert_allclose(c, arr[name + "_c"], rtol=0, atol=1e-13, err_msg=name)


def test_loop_core_equals_vector_core():
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal(60), rng.standard_normal(60)
    c1 = rng.standard_normal(40)
    c2 = c1.copy()
    gemm_core(4, 5, 3, 1.5, a, 2, 1, 7, b, 1, 1, 4, 0.5, c1, 3, 1, 6)
    gemm_core_loops(4, 5, 3, 1.5, a, 2, 1, 7, b, 1, 1, 4, 0.5, c2, 3, 1, 6)
    np.testing.assert_allclose(c1, c2, atol=1e-14)


def test_beta_zero_never_reads_c():
    a = np.ones(4)
    c = np.full(4, np.nan)
    batched_core(2, 2, 2, 1.0, a, 0, 1, 2, 0, a, 0, 1, 2, 0, 0.0, c, 0, 1, 2, 0, 1)
    np.testing.assert_array_equal(c, np.full(4, 2.0))


@pytest.mark.parametrize("idx", range(5))
def test_oracle_hooi_matches_reference(golden_hooi, idx):
    index, arr = golden_hooi
    rec = index["records"][idx]
    name = rec["name"]
    t = arr[name + "_t"].reshape(rec["dims"], order="F")
    got = otucker.hooi(t, rec["ranks"], max_iters=rec["max_iters"])
    # fit = 1 - sqrt(max(0, |T|^2 - |G|^2))/|T| (tucker.py:164-167) turns a 1e-16
    # cancellation into ~1e-8, so at exact rank the early-stop iteration can move by one.
    assert abs(got["iterations"] - rec["iterations"]) <= (1 if rec["fit_history"][-1] > 0.999999 else 0)
    nfit = min(len(got["fit_history"]), len(rec["fit_history"]))
    np.testing.assert_allclose(got["fit_history"][:nfit], rec["fit_history"][:nfit], rtol=0, atol=1e-7)
    for r in range(3):
        u_ref = arr[f"{name}_u{r}"]
        u = got["factors"][r]
        # same subspace, same sign convention
        np.testing.assert_allclose(u @ u.T, u_ref @ u_ref.T, atol=1e-7)
    rec_t = otucker.reconstruct(got["core"], got["factors"])
    np.testing.assert_allclose(rec_t.reshape(-1, order="F"), arr[name + "_rec"], atol=1e-7)
