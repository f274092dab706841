"""The conventional (permute-then-GEMM) comparison strategy: plans must equal
the reference's plan_conventional (planner.py:411-465) and device execution
must reproduce contract_conventional's outputs and counters
(planner.py:620-713, reference.py:54-63) -- golden fixtures from the real
reference (tests/golden/conventional.*)."""
import numpy as np
import pytest

from conftest import GOLDEN, load_json
from paper_1606_05696_b200.layout import Layout
from paper_1606_05696_b200.notation import ContractionSpec
from paper_1606_05696_b200.planner import PermuteStep, plan_conventional


@pytest.fixture(scope="module")
def golden_all():
    return load_json("conventional.json")["records"], np.load(GOLDEN / "conventional.npz")


@pytest.fixture(scope="module")
def golden_conv(golden_all):
    records, arr = golden_all
    return [r for r in records if r["policy"] != "batched-gemv"], arr


@pytest.fixture(scope="module")
def golden_gemv(golden_all):
    records, arr = golden_all
    return [r for r in records if r["policy"] == "batched-gemv"], arr


def _plan(rec):
    spec = ContractionSpec(tuple(rec["a"]), tuple(rec["b"]), tuple(rec["c"]),
                           alpha=rec["alpha"], beta=rec["beta"])
    ext = rec["ext"]
    lays = [Layout.packed([ext[l] for l in labs]) for labs in (rec["a"], rec["b"], rec["c"])]
    return spec, lays, plan_conventional(spec, *lays, policy=rec["policy"])


def test_conventional_plans_match_reference(golden_conv):
    records, _ = golden_conv
    assert len(records) == 36 * 2 * 2
    for rec in records:
        _, _, plan = _plan(rec)
        info = plan.conventional
        assert plan.strategy == "conventional"
        assert [[s.tensor, list(s.perm)] for s in plan.steps
                if isinstance(s, PermuteStep)] == rec["steps"], rec["key"]
        assert plan.predicted_transpositions == rec["predicted_transpositions"], rec["key"]
        assert (info.op_a.value, info.op_b.value) == (rec["op_a"], rec["op_b"]), rec["key"]
        assert (None if info.permute_a is None else list(info.permute_a)) == rec["permute_a"]
        assert (None if info.permute_b is None else list(info.permute_b)) == rec["permute_b"]
        assert info.c_matches == rec["c_matches"] and info.family == rec["family"]


def test_conventional_rejects_unknown_policy():
    spec = ContractionSpec(tuple("mk"), tuple("knp"), tuple("mnp"))
    lays = [Layout.packed((2, 3)), Layout.packed((3, 4, 5)), Layout.packed((2, 4, 5))]
    with pytest.raises(ValueError):
        plan_conventional(spec, *lays, policy="fast")


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_conventional_execution_matches_reference(golden_conv, dtype):
    import torch

    import paper_1606_05696_b200 as sbt
    from paper_1606_05696_b200.layout import DenseTensor
    from oracle import naive
    records, arr = golden_conv
    tdt = torch.float64 if dtype == "float64" else torch.float32
    tol = 1e-12 if dtype == "float64" else 1e-5
    for rec in records:
        spec, lays, _ = _plan(rec)
        key = rec["key"]
        a = DenseTensor(lays[0], torch.as_tensor(arr[key + "_a"], device="cuda").to(tdt))
        b = DenseTensor(lays[1], torch.as_tensor(arr[key + "_b"], device="cuda").to(tdt))
        c = DenseTensor(lays[2], torch.as_tensor(arr[key + "_c0"], device="cuda").to(tdt))
        counters = sbt.contract_conventional(spec, a, b, rec["alpha"], rec["beta"], c,
                                             policy=rec["policy"])
        got = c.data.double().cpu().numpy()
        if dtype == "float64":
            want = arr[key + "_c"]
        else:  # fp32 inputs: fp64 reference arithmetic on the fp32-rounded values
            from oracle import plan as oplan
            want = c.data.new_tensor(arr[key + "_c0"]).double().cpu().numpy().copy()
            oplan.contract(tuple(rec["a"]), tuple(rec["b"]), tuple(rec["c"]), rec["ext"],
                           a.data.double().cpu().numpy(), b.data.double().cpu().numpy(),
                           rec["alpha"], rec["beta"], want)
        assert naive.max_rel_err(got, want) <= tol, key
        assert counters.transpositions == rec["transpositions"], key
        assert counters.kernel_calls == rec["kernel_calls"], key


@pytest.mark.gpu
def test_permute_copy_matches_numpy():
    import itertools

    import torch

    from paper_1606_05696_b200.layout import DenseTensor, permute_copy, transposition_count
    rng = np.random.default_rng(3)
    for dims in ((5, 7, 3), (64, 33, 40), (1, 9, 130), (17, 1, 31, 6)):
        x = rng.uniform(-1, 1, dims)
        t = DenseTensor.from_array(x)
        for perm in itertools.permutations(range(len(dims))):
            n0 = transposition_count()
            out = permute_copy(t, perm)
            torch.cuda.synchronize()
            assert transposition_count() == n0 + 1
            np.testing.assert_array_equal(out.to_array(), np.transpose(x, perm))


# ------------------------------------------------------------------ batched-GEMV strategy


def _gemv_plan(rec):
    from paper_1606_05696_b200.planner import plan_batched_gemv
    spec = ContractionSpec(tuple(rec["a"]), tuple(rec["b"]), tuple(rec["c"]))
    ext = rec["ext"]
    lays = [Layout.packed([ext[l] for l in labs]) for labs in (rec["a"], rec["b"], rec["c"])]
    return spec, lays, plan_batched_gemv(spec, *lays)


def test_batched_gemv_plans_match_reference(golden_gemv):
    from paper_1606_05696_b200.planner import FlattenStep, GemvBatchStep
    records, _ = golden_gemv
    assert len(records) == 36 * 2
    for rec in records:
        _, _, plan = _gemv_plan(rec)
        assert plan.strategy == "batched-gemv"
        st = plan.steps[-1]
        assert isinstance(st, GemvBatchStep)
        assert {"loop_labels": list(st.loop_labels), "matrix": st.matrix, "op": st.op.value,
                "v_label": st.v_label, "k_label": st.k_label} == rec["gemv"], rec["key"]
        assert [[f.tensor, list(f.labels), f.merged] for f in plan.steps
                if isinstance(f, FlattenStep)] == rec["flatten"], rec["key"]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_batched_gemv_execution_matches_reference(golden_gemv, dtype):
    import torch

    from paper_1606_05696_b200 import _lib
    from paper_1606_05696_b200.layout import DenseTensor
    from paper_1606_05696_b200.planner import execute_plan
    from oracle import naive, plan as oplan
    records, arr = golden_gemv
    tdt = torch.float64 if dtype == "float64" else torch.float32
    tol = 1e-12 if dtype == "float64" else 1e-5
    for rec in records:
        spec, lays, plan = _gemv_plan(rec)
        key = rec["key"]
        a = DenseTensor(lays[0], torch.as_tensor(arr[key + "_a"], device="cuda").to(tdt))
        b = DenseTensor(lays[1], torch.as_tensor(arr[key + "_b"], device="cuda").to(tdt))
        c = DenseTensor(lays[2], torch.as_tensor(arr[key + "_c0"], device="cuda").to(tdt))
        n0 = _lib.launch_count()
        execute_plan(plan, a, b, rec["alpha"], rec["beta"], c)
        assert _lib.launch_count() - n0 == 1, key      # every GEMV of the loop in one launch
        assert _lib.last_kernel().startswith("gemv_"), _lib.last_kernel()
        got = c.data.double().cpu().numpy()
        if dtype == "float64":
            want = arr[key + "_c"]
        else:
            want = c.data.new_tensor(arr[key + "_c0"]).double().cpu().numpy().copy()
            oplan.contract(tuple(rec["a"]), tuple(rec["b"]), tuple(rec["c"]), rec["ext"],
                           a.data.double().cpu().numpy(), b.data.double().cpu().numpy(),
                           rec["alpha"], rec["beta"], want)
        assert naive.max_rel_err(got, want) <= tol, key
