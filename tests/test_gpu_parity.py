"""Parity of the sm_100a path against the reference (golden fixtures) and the
CPU oracle.  Tolerances (north_star): max_rel_err <= 1e-12 for fp64, <= 1e-5
for fp32 (fp32 results are checked against an fp64 oracle run on the same
fp32 values)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1606_05696_b200 as sbt  # noqa: E402
from paper_1606_05696_b200 import _lib, backend, kernels, layout as L  # noqa: E402
from paper_1606_05696_b200.kernels import Op  # noqa: E402
from paper_1606_05696_b200.layout import DenseTensor, Layout  # noqa: E402
from paper_1606_05696_b200.notation import ContractionSpec  # noqa: E402
from paper_1606_05696_b200.planner import (BatchedStep, enumerate_cases, execute_plan,  # noqa: E402
                                           find_case, plan_single_mode)
from oracle import api as oapi, naive, plan as oplan  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = {torch.float64: 1e-12, torch.float32: 1e-5}
EXCEPTIONAL = {"3.4", "3.6", "4.4", "4.6", "5.4", "5.6", "6.4", "6.6"}


def dev(x, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(x)).to(device="cuda", dtype=dtype)


def host(t):
    return t.detach().double().cpu().numpy()


@pytest.fixture(autouse=True)
def _auto_kernels():
    _lib.set_kernel_override("auto")
    yield
    _lib.set_kernel_override("auto")


def _packed(spec, ext):
    return (Layout.packed([ext[l] for l in spec.labels_a]),
            Layout.packed([ext[l] for l in spec.labels_b]),
            Layout.packed([ext[l] for l in spec.labels_c] or [1]))


# ------------------------------------------------------------------ golden fixtures


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_all_36_cases_match_reference_outputs(golden_contract, dtype):
    index, arr = golden_contract
    for rec in index["records"]:
        key = rec["key"]
        spec = ContractionSpec(tuple(rec["a"]), tuple(rec["b"]), tuple(rec["c"]))
        la, lb, lc = _packed(spec, rec["ext"])
        a = DenseTensor(la, dev(arr[key + "_a"], dtype))
        b = DenseTensor(lb, dev(arr[key + "_b"], dtype))
        c = DenseTensor(lc, dev(arr[key + "_c0"], dtype))
        execute_plan(plan_single_mode(spec, la, lb, lc), a, b, rec["alpha"], rec["beta"], c)
        if dtype == torch.float64:
            want = arr[key + "_c"]
        else:  # fp64 oracle on the fp32-rounded inputs
            want = host(c.data) * 0
            want[:] = host(dev(arr[key + "_c0"], dtype))
            oplan.contract(rec["a"], rec["b"], rec["c"], rec["ext"],
                           host(dev(arr[key + "_a"], dtype)), host(dev(arr[key + "_b"], dtype)),
                           rec["alpha"], rec["beta"], want)
        err = naive.max_rel_err(host(c.data), want)
        assert err <= TOL[dtype], (key, err)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_kernel_entry_points_match_reference(golden_kernels, dtype):
    index, arr = golden_kernels
    for rec in index["records"]:
        name, kw = rec["name"], dict(rec["kw"])
        a, b = dev(arr[name + "_a"], dtype), dev(arr[name + "_b"], dtype)
        c = dev(arr[name + "_c0"], dtype)
        getattr(kernels, rec["fn"])(a=a, b=b, c=c, **kw)
        if dtype == torch.float64:
            want = arr[name + "_c"]
        else:
            want = host(dev(arr[name + "_c0"], dtype))
            oapi.run_call(rec["fn"], kw, host(a), host(b), want)
        assert naive.max_rel_err(host(c), want) <= TOL[dtype], name


def test_numpy_buffers_take_the_host_seam(golden_kernels):
    index, arr = golden_kernels
    for rec in index["records"]:
        name = rec["name"]
        c = arr[name + "_c0"].copy()
        getattr(kernels, rec["fn"])(a=arr[name + "_a"].copy(), b=arr[name + "_b"].copy(), c=c,
                                    **rec["kw"])
        assert naive.max_rel_err(c, arr[name + "_c"]) <= 1e-12, name


def test_backend_adapter_reference_signatures(golden_kernels):
    index, arr = golden_kernels
    for rec in index["records"]:
        name = rec["name"]
        cl = oapi.lower_call(rec["fn"], rec["kw"])
        c = arr[name + "_c0"].copy()
        backend.batched_core(cl["m"], cl["n"], cl["k"], rec["kw"]["alpha"], arr[name + "_a"],
                             cl["oa"], cl["ars"], cl["acs"], cl["apt"], arr[name + "_b"], cl["ob"],
                             cl["brs"], cl["bcs"], cl["bpt"], rec["kw"]["beta"], c, cl["oc"],
                             cl["crs"], cl["ccs"], cl["cpt"], cl["batch"])
        assert naive.max_rel_err(c, arr[name + "_c"]) <= 1e-12, name


def test_host_seam_preserves_gaps_in_c():
    rng = np.random.default_rng(7)
    m, n, k, P = 3, 4, 5, 6
    a, b = rng.standard_normal(m * k * P), rng.standard_normal(k * n * P)
    c = rng.standard_normal(2 * m * n * P)       # ldc = 2m: every other column is a gap
    want = c.copy()
    oapi.run_call("strided_batched_gemm", dict(opa="N", opb="N", m=m, n=n, k=k, alpha=1.0,
                  lda=m, loa=m * k, ldb=k, lob=k * n, beta=0.0, ldc=2 * m, loc=2 * m * n,
                  batch_count=P), a, b, want)
    kernels.strided_batched_gemm("N", "N", m, n, k, 1.0, a, m, m * k, b, k, k * n, 0.0, c,
                                 2 * m, 2 * m * n, P)
    np.testing.assert_allclose(c, want, rtol=0, atol=1e-13)


# ------------------------------------------------------------------ reference semantics


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_beta_zero_ignores_nan(dtype):
    c = torch.full((4,), float("nan"), dtype=dtype, device="cuda")
    one = torch.ones(4, dtype=dtype, device="cuda")
    kernels.gemm(Op.Normal, Op.Normal, 2, 2, 2, 1.0, one, 2, one, 2, 0.0, c, 2)
    assert torch.equal(c.cpu(), torch.full((4,), 2.0, dtype=dtype))


def test_batch_zero_and_broadcast():
    c = torch.full((8,), 5.0, dtype=torch.float64, device="cuda")
    z = torch.zeros(8, dtype=torch.float64, device="cuda")
    n0 = _lib.launch_count()
    kernels.strided_batched_gemm(Op.Normal, Op.Normal, 2, 2, 2, 1.0, z, 2, 4, z, 2, 4, 0.0, c,
                                 2, 4, 0)
    assert _lib.launch_count() == n0
    assert torch.equal(c.cpu(), torch.full((8,), 5.0, dtype=torch.float64))
    rng = np.random.default_rng(3)
    m, n, k, P = 3, 4, 2, 5
    A = rng.standard_normal((m, k, P))
    B = rng.standard_normal((k, n))
    c = torch.zeros(m * n * P, dtype=torch.float64, device="cuda")
    kernels.strided_batched_gemm(Op.Normal, Op.Normal, m, n, k, 1.0,
                                 dev(A.reshape(-1, order="F")), m, m * k,
                                 dev(B.reshape(-1, order="F")), k, 0, 0.0, c, m, m * n, P)
    want = np.einsum("ikp,kn->inp", A, B)
    np.testing.assert_allclose(host(c).reshape((m, n, P), order="F"), want, atol=1e-13)


def test_extended_equals_per_batch_loop():
    rng = np.random.default_rng(4)
    for exop in (Op.ExtendedNormal, Op.ExtendedTranspose):
        m, n, k, P = 3, 4, 2, 5
        a = dev(rng.standard_normal(P * m * k + 7))
        b = dev(rng.standard_normal(max(k, n) ** 2 + 40))
        lda, loa = (P, P * m) if exop is Op.ExtendedNormal else (P, P * k)
        c1 = torch.zeros(m * n * P, dtype=torch.float64, device="cuda")
        c2 = torch.zeros_like(c1)
        args = (exop, Op.Normal, m, n, k, 1.0, a, lda, loa, b, k, 0, 0.0)
        kernels.strided_batched_gemm_ex(*args, c1, m, m * n, P)
        kernels.strided_batched_gemm_ex_reference(*args, c2, m, m * n, P)
        assert naive.max_rel_err(host(c1), host(c2)) <= 1e-15


def test_extended_matches_permute_then_batched():
    rng = np.random.default_rng(3)
    for cid in sorted(EXCEPTIONAL):
        case = find_case(2, 3, cid)
        spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
        ext = {l: int(rng.integers(2, 9)) for l in "mnpk"}
        la, lb, lc = _packed(spec, ext)
        A = rng.uniform(-1, 1, la.dims)
        Bt = rng.uniform(-1, 1, lb.dims)
        a, b = DenseTensor.from_array(A), DenseTensor.from_array(Bt)
        c = DenseTensor.zeros(lc)
        plan = plan_single_mode(spec, la, lb, lc)
        step = plan.steps[-1]
        assert isinstance(step, BatchedStep) and step.extended
        execute_plan(plan, a, b, 1.0, 0.0, c)
        first = step.gemm.first
        labels_x = spec.labels_a if first == "A" else spec.labels_b
        X = A if first == "A" else Bt
        pos = labels_x.index(step.batch_label)
        perm = [i for i in range(len(labels_x)) if i != pos] + [pos]
        x2 = DenseTensor.from_array(np.transpose(X, perm))
        lx2 = tuple(labels_x[i] for i in perm)
        spec2 = (ContractionSpec(lx2, spec.labels_b, spec.labels_c) if first == "A"
                 else ContractionSpec(spec.labels_a, lx2, spec.labels_c))
        a2, b2 = (x2, b) if first == "A" else (a, x2)
        c2 = DenseTensor.zeros(lc)
        plan2 = plan_single_mode(spec2, a2.layout, b2.layout, c2.layout)
        assert plan2.strategy != "extended-batched"
        execute_plan(plan2, a2, b2, 1.0, 0.0, c2)
        assert naive.max_rel_err(c.host_data(), c2.host_data()) <= 1e-13, cid


def test_zero_copies_and_one_launch_per_plan():
    rng = np.random.default_rng(2)
    ext = dict(m=5, n=4, p=6, k=3)
    for case in enumerate_cases(2, 3):
        spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
        la, lb, lc = _packed(spec, ext)
        a = DenseTensor.from_array(rng.uniform(-1, 1, la.dims))
        b = DenseTensor.from_array(rng.uniform(-1, 1, lb.dims))
        c = DenseTensor.zeros(lc)
        plan = plan_single_mode(spec, la, lb, lc)
        assert plan.predicted_transpositions == 0
        t0, a0, n0 = L.transposition_count(), L.allocation_count(), _lib.launch_count()
        torch.cuda.synchronize()
        mem0 = torch.cuda.memory_allocated()
        execute_plan(plan, a, b, 1.0, 0.0, c)
        torch.cuda.synchronize()
        assert (L.transposition_count(), L.allocation_count()) == (t0, a0), case.case_id
        assert torch.cuda.memory_allocated() == mem0
        assert _lib.launch_count() == n0 + 1, case.case_id


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_zero_copies_at_bench_size(dtype):
    """The n = 256 sweep extents (every case, both dtypes): no transposition, no
    tensor allocation, no growth of the caching allocator, one launch per
    planned contraction -- the device memory the kernels see is the caller's."""
    n = 256
    g = torch.Generator(device="cuda").manual_seed(5)
    a2 = torch.rand(n * n, generator=g, device="cuda", dtype=dtype)
    b3 = torch.rand(n ** 3, generator=g, device="cuda", dtype=dtype)
    c3 = torch.empty(n ** 3, device="cuda", dtype=dtype)
    for case in enumerate_cases(2, 3):
        spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
        la, lb, lc = _packed(spec, dict(m=n, n=n, p=n, k=n))
        a = DenseTensor(la, a2 if la.size == n * n else b3)
        b = DenseTensor(lb, a2 if lb.size == n * n else b3)
        c = DenseTensor(lc, c3)
        plan = plan_single_mode(spec, la, lb, lc)
        execute_plan(plan, a, b, 1.0, 0.0, c)      # first call: tensor maps, attributes
        torch.cuda.synchronize()
        t0, a0, n0 = L.transposition_count(), L.allocation_count(), _lib.launch_count()
        mem0 = torch.cuda.memory_allocated()
        execute_plan(plan, a, b, 1.0, 0.0, c)
        torch.cuda.synchronize()
        assert (L.transposition_count(), L.allocation_count()) == (t0, a0), case.case_id
        assert torch.cuda.memory_allocated() == mem0, case.case_id
        assert _lib.launch_count() == n0 + 1, case.case_id


def test_nested_batching_single_launch():
    rng = np.random.default_rng(4)
    spec = ContractionSpec(tuple("mkp"), tuple("nkq"), tuple("mnpq"))
    for p, q in ((4, 7), (7, 4)):
        ext = dict(m=5, n=6, k=3, p=p, q=q)
        la, lb, lc = _packed(spec, ext)
        A, B = rng.uniform(-1, 1, la.dims), rng.uniform(-1, 1, lb.dims)
        a, b, c = DenseTensor.from_array(A), DenseTensor.from_array(B), DenseTensor.zeros(lc)
        n0 = _lib.launch_count()
        execute_plan(plan_single_mode(spec, la, lb, lc), a, b, 1.0, 0.0, c)
        assert _lib.launch_count() == n0 + 1
        want = np.einsum("mkp,nkq->mnpq", A, B)
        assert naive.max_rel_err(c.to_array(), want) <= 1e-12


def test_aliased_output_and_drift_rejected():
    spec = sbt.parse_contraction("C[mn] = A[mk] * B[kn]")
    a = DenseTensor.from_array(np.ones((3, 3)))
    b = DenseTensor.from_array(np.ones((3, 3)))
    c = DenseTensor.zeros((3, 3))
    plan = plan_single_mode(spec, a.layout, b.layout, c.layout)
    with pytest.raises(sbt.PlanError):
        execute_plan(plan, a, b, 1.0, 0.0, DenseTensor(c.layout, a.data))
    with pytest.raises(sbt.PlanError):
        execute_plan(plan, a, b, 1.0, 0.0, DenseTensor.zeros((3, 4)))


def test_scalar_output_dot():
    rng = np.random.default_rng(5)
    spec = ContractionSpec(("k",), ("k",), ())
    x, y = rng.uniform(-1, 1, 7), rng.uniform(-1, 1, 7)
    a, b = DenseTensor.from_array(x), DenseTensor.from_array(y)
    c = DenseTensor.zeros((1,))
    execute_plan(plan_single_mode(spec, a.layout, b.layout, c.layout), a, b, 2.0, 0.0, c)
    assert abs(c.host_data()[0] - 2.0 * x @ y) <= 1e-13


# ------------------------------------------------------------------ larger sizes vs oracle


def _case_run(cid, n, dtype, seed, alpha=1.0, beta=0.0):
    rng = np.random.default_rng(seed)
    case = find_case(2, 3, cid)
    spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
    ext = dict(m=n, n=n, p=n, k=n)
    la, lb, lc = _packed(spec, ext)
    ha = rng.uniform(-1, 1, la.size)
    hb = rng.uniform(-1, 1, lb.size)
    hc = rng.uniform(-1, 1, lc.size)
    a = DenseTensor(la, dev(ha, dtype))
    b = DenseTensor(lb, dev(hb, dtype))
    c = DenseTensor(lc, dev(hc, dtype))
    execute_plan(plan_single_mode(spec, la, lb, lc), a, b, alpha, beta, c)
    want = host(dev(hc, dtype)).copy()
    oplan.contract(spec.labels_a, spec.labels_b, spec.labels_c, ext, host(a.data),
                   host(b.data), alpha, beta, want)
    return naive.max_rel_err(host(c.data), want)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("n", [64, 128])
def test_36_cases_square_vs_oracle(n, dtype):
    for i, case in enumerate(enumerate_cases(2, 3)):
        err = _case_run(case.case_id, n, dtype, seed=1000 * n + i, alpha=1.25,
                        beta=0.5 if i % 3 == 0 else 0.0)
        assert err <= TOL[dtype], (case.case_id, n, err)


@pytest.mark.parametrize("which", ["generic", "auto"])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_kernel_families_agree_on_odd_and_aligned_shapes(which, dtype):
    _lib.set_kernel_override(which)
    rng = np.random.default_rng(11)
    for (m, n, k, P) in ((7, 5, 3, 9), (33, 17, 65, 4), (128, 96, 64, 3), (256, 256, 128, 2)):
        for opa in ("N", "T"):
            for opb in ("N", "T"):
                lda = m if opa == "N" else k
                ldb = k if opb == "N" else n
                ha, hb = rng.uniform(-1, 1, m * k * P), rng.uniform(-1, 1, k * n * P)
                c = torch.zeros(m * n * P, dtype=dtype, device="cuda")
                a, b = dev(ha, dtype), dev(hb, dtype)
                kernels.strided_batched_gemm(opa, opb, m, n, k, 1.0, a, lda, m * k, b, ldb, k * n,
                                             0.0, c, m, m * n, P)
                want = np.zeros(m * n * P)
                oapi.run_call("strided_batched_gemm", dict(opa=opa, opb=opb, m=m, n=n, k=k,
                              alpha=1.0, lda=lda, loa=m * k, ldb=ldb, lob=k * n, beta=0.0,
                              ldc=m, loc=m * n, batch_count=P), host(a), host(b), want)
                assert naive.max_rel_err(host(c), want) <= TOL[dtype], (m, n, k, P, opa, opb)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("n", [8, 16, 32, 64])
def test_small_matrix_batches(n, dtype):
    rng = np.random.default_rng(n)
    P = 2000
    ha, hb = rng.uniform(-1, 1, n * n * P), rng.uniform(-1, 1, n * n * P)
    a, b = dev(ha, dtype), dev(hb, dtype)
    c = torch.zeros(n * n * P, dtype=dtype, device="cuda")
    kernels.strided_batched_gemm("N", "N", n, n, n, 1.0, a, n, n * n, b, n, n * n, 0.0, c, n,
                                 n * n, P)
    want = np.matmul(host(a).reshape(P, n, n).transpose(0, 2, 1),
                     host(b).reshape(P, n, n).transpose(0, 2, 1)).transpose(0, 2, 1).reshape(-1)
    assert naive.max_rel_err(host(c), want) <= TOL[dtype]


# ------------------------------------------------------------------ Tucker / HOOI


@pytest.mark.parametrize("idx", range(5))
def test_hooi_matches_reference_fp64(golden_hooi, idx):
    index, arr = golden_hooi
    rec = index["records"][idx]
    name = rec["name"]
    t = DenseTensor(Layout.packed(rec["dims"]), dev(arr[name + "_t"]))
    model = sbt.hooi(t, rec["ranks"], max_iters=rec["max_iters"])
    if rec["fit_history"][-1] < 0.999999:
        assert model.iterations == rec["iterations"]
    else:
        # exact rank: fit = 1 - sqrt(max(0,|T|^2-|G|^2))/|T| turns 1e-16 cancellation
        # noise into ~1e-8 wobble, so the early-stop iteration is noise-driven
        assert model.iterations <= rec["max_iters"]
    nf = min(len(model.fit_history), len(rec["fit_history"]))
    np.testing.assert_allclose(model.fit_history[:nf], rec["fit_history"][:nf], atol=1e-7)
    for r in range(3):
        u = model.factors[r].cpu().numpy()
        ur = arr[f"{name}_u{r}"]
        np.testing.assert_allclose(u @ u.T, ur @ ur.T, atol=1e-7)
        np.testing.assert_allclose(u.T @ u, np.eye(u.shape[1]), atol=1e-10)
    rec_t = sbt.tucker_reconstruct(model)
    np.testing.assert_allclose(rec_t.host_data(), arr[name + "_rec"], atol=1e-7)


def test_hooi_fp32_matches_oracle():
    from oracle import tucker as otucker
    rng = np.random.default_rng(9)
    dims, ranks = (64, 48, 40), (6, 5, 4)
    core = rng.standard_normal(ranks)
    us = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
    full = np.einsum("abc,ia,jb,kc->ijk", core, *us) + 1e-3 * rng.standard_normal(dims)
    t = DenseTensor.from_array(full, dtype="float32")
    model = sbt.hooi(t, ranks, max_iters=4, tol=-1.0)
    ref = otucker.hooi(t.to_array().astype(np.float64), ranks, max_iters=4, tol=-1.0)
    np.testing.assert_allclose(model.fit_history, ref["fit_history"], rtol=1e-5)
    for r in range(3):
        u = model.factors[r].cpu().numpy()
        ur = ref["factors"][r]
        np.testing.assert_allclose(u @ u.T, ur @ ur.T, atol=1e-4)


# ------------------------------------------------------------------ kernel families / paths


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_small_matrix_kernel_forced_layouts(dtype):
    """K3 on every dense storage order, odd and multiple-of-4 extents, beta != 0."""
    _lib.set_kernel_override("small")
    rng = np.random.default_rng(21)
    for (m, n, k, P) in ((8, 8, 8, 300), (12, 16, 4, 257), (32, 32, 32, 70), (6, 10, 14, 50),
                         (64, 64, 64, 5)):
        for opa in ("N", "T"):
            for opb in ("N", "T"):
                lda = m if opa == "N" else k
                ldb = k if opb == "N" else n
                ha, hb = rng.uniform(-1, 1, m * k * P), rng.uniform(-1, 1, k * n * P)
                hc = rng.uniform(-1, 1, m * n * P)
                a, b, c = dev(ha, dtype), dev(hb, dtype), dev(hc, dtype)
                kernels.strided_batched_gemm(opa, opb, m, n, k, 0.75, a, lda, m * k, b, ldb,
                                             k * n, -0.5, c, m, m * n, P)
                want = host(dev(hc, dtype)).copy()
                oapi.run_call("strided_batched_gemm", dict(opa=opa, opb=opb, m=m, n=n, k=k,
                              alpha=0.75, lda=lda, loa=m * k, ldb=ldb, lob=k * n, beta=-0.5,
                              ldc=m, loc=m * n, batch_count=P), host(a), host(b), want)
                got = _lib.last_kernel()
                assert naive.max_rel_err(host(c), want) <= TOL[dtype], (m, n, k, opa, opb, got)


def test_split_k_for_tall_reductions():
    rng = np.random.default_rng(5)
    for dtype in (torch.float64, torch.float32):
        m, n, k = 96, 64, 70000
        ha, hb = rng.uniform(-1, 1, m * k), rng.uniform(-1, 1, k * n)
        a, b = dev(ha, dtype), dev(hb, dtype)
        c = torch.zeros(m * n, dtype=dtype, device="cuda")
        n0 = _lib.launch_count()
        kernels.gemm("N", "N", m, n, k, 1.0, a, m, b, k, 0.0, c, m)
        if dtype == torch.float64:   # narrow N: the skinny kernel reduces its splits in-kernel
            assert _lib.last_kernel() == "skinny_dmma_f64", _lib.last_kernel()
        else:
            assert _lib.launch_count() - n0 >= 2  # split partials + reduction
        want = np.zeros(m * n)
        oapi.run_call("gemm", dict(opa="N", opb="N", m=m, n=n, k=k, alpha=1.0, lda=m, ldb=k,
                      beta=0.0, ldc=m), host(a), host(b), want)
        assert naive.max_rel_err(host(c), want) <= TOL[dtype] * 4


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_fourth_order_nested_single_launch_n64(dtype):
    rng = np.random.default_rng(8)
    spec = ContractionSpec(tuple("mkp"), tuple("nkq"), tuple("mnpq"))
    ext = dict(m=64, n=48, k=32, p=40, q=24)
    la, lb, lc = _packed(spec, ext)
    A, B = rng.uniform(-1, 1, la.dims), rng.uniform(-1, 1, lb.dims)
    a, b = DenseTensor.from_array(A, dtype=dtype), DenseTensor.from_array(B, dtype=dtype)
    c = DenseTensor.zeros(lc, dtype=dtype)
    n0 = _lib.launch_count()
    execute_plan(plan_single_mode(spec, la, lb, lc), a, b, 1.0, 0.0, c)
    assert _lib.launch_count() == n0 + 1
    want = np.einsum("mkp,nkq->mnpq", a.to_array().astype(np.float64),
                     b.to_array().astype(np.float64))
    assert naive.max_rel_err(c.to_array(), want) <= TOL[dtype]


def test_hooi_mode0_reuse_is_bitwise_identical():
    rng = np.random.default_rng(13)
    dims, ranks = (40, 36, 32), (5, 4, 3)
    core = rng.standard_normal(ranks)
    us = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
    full = np.einsum("abc,ia,jb,kc->ijk", core, *us) + 1e-2 * rng.standard_normal(dims)
    for dtype in ("float32", "float64"):
        t = DenseTensor.from_array(full, dtype=dtype)
        m1 = sbt.hooi(t, ranks, max_iters=3, tol=-1.0, reuse_mode0=True)
        m2 = sbt.hooi(t, ranks, max_iters=3, tol=-1.0, reuse_mode0=False)
        assert m1.fit_history == m2.fit_history
        for u1, u2 in zip(m1.factors, m2.factors):
            assert torch.equal(u1, u2)
        assert torch.equal(m1.core.data, m2.core.data)


def test_tensor_paths_are_used_for_the_36_cases():
    """No silent fallback: at n=64 every case runs on a tensor-core kernel."""
    rng = np.random.default_rng(1)
    for dtype, prefix in ((torch.float32, ("tc_tf32x3",)),
                          (torch.float64, ("tc_dmma", "skinny_dmma"))):
        for case in enumerate_cases(2, 3):
            spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
            la, lb, lc = _packed(spec, dict(m=64, n=64, p=64, k=64))
            a = DenseTensor(la, dev(rng.uniform(-1, 1, la.size), dtype))
            b = DenseTensor(lb, dev(rng.uniform(-1, 1, lb.size), dtype))
            c = DenseTensor(lc, torch.empty(lc.size, dtype=dtype, device="cuda"))
            execute_plan(plan_single_mode(spec, la, lb, lc), a, b, 1.0, 0.0, c)
            assert _lib.last_kernel().startswith(prefix), (case.case_id, _lib.last_kernel())


def test_fp64_probe_reports_a_plausible_peak():
    tf = _lib.probe_fp64_peak("dmma")
    assert 5.0 < tf < 100.0


# ------------------------------------------------------------------ exceptional cases, batch-blocked


def _strided_case_run(cid, ext, pad, dtype, seed, alpha=1.0, beta=0.0):
    """One case with the 3rd-order operand's first mode padded to ``pad``
    elements (leading dimension > extent): ragged batch groups, non-packed."""
    rng = np.random.default_rng(seed)
    case = find_case(2, 3, cid)
    spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)

    def lay(labels, padded):
        dims = [ext[l] for l in labels]
        strides, s = [], 1
        for i, d in enumerate(dims):
            strides.append(s)
            s *= (pad if (padded and i == 0) else d)
        return Layout(tuple(dims), tuple(strides))

    la = lay(spec.labels_a, len(spec.labels_a) == 3)
    lb = lay(spec.labels_b, len(spec.labels_b) == 3)
    lc = Layout.packed([ext[l] for l in spec.labels_c])
    ha = rng.uniform(-1, 1, la.min_buffer_len())
    hb = rng.uniform(-1, 1, lb.min_buffer_len())
    hc = rng.uniform(-1, 1, lc.size)
    a, b = DenseTensor(la, dev(ha, dtype)), DenseTensor(lb, dev(hb, dtype))
    c = DenseTensor(lc, dev(hc, dtype))
    execute_plan(plan_single_mode(spec, la, lb, lc), a, b, alpha, beta, c)
    kern = _lib.last_kernel()
    want = host(dev(hc, dtype)).copy()
    oplan.contract(spec.labels_a, spec.labels_b, spec.labels_c, ext, host(a.data),
                   host(b.data), alpha, beta, want, layouts=(la, lb, lc))
    return naive.max_rel_err(host(c.data), want), kern


@pytest.mark.parametrize("cid", sorted(EXCEPTIONAL))
def test_exceptional_cases_batch_blocked_f64_n256(cid):
    """fp64 exceptional cases on the batch-blocked DMMA tiles."""
    err = _case_run(cid, 256, torch.float64, seed=5 + hash(cid) % 89, alpha=-1.25, beta=0.5)
    assert _lib.last_kernel() == "tc_dmma_f64_bb", (cid, _lib.last_kernel())
    assert err <= TOL[torch.float64], (cid, err)


@pytest.mark.parametrize("cid", sorted(EXCEPTIONAL))
def test_exceptional_cases_batch_blocked_n256(cid):
    """fp32 exceptional cases run on the batch-blocked CTA-pair kernel (A's
    unit-stride batch folded into the MMA rows) and match the oracle."""
    err = _case_run(cid, 256, torch.float32, seed=7 + hash(cid) % 97, alpha=0.75, beta=0.5)
    assert err <= TOL[torch.float32], (cid, err)
    err = _case_run(cid, 256, torch.float32, seed=3)
    assert _lib.last_kernel().startswith("tc_tf32x3_pair_bb"), (cid, _lib.last_kernel())
    assert err <= TOL[torch.float32], (cid, err)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("cid", ["3.4", "4.6", "5.6", "6.4"])
def test_exceptional_ragged_batch_groups(cid, dtype):
    """Batch extent not a multiple of 4 (padded leading dimension), ragged
    m / n / k tails: the batch-blocked tiles must mask rows and zero-fill."""
    case = find_case(2, 3, cid)
    third, second = ((case.labels_b, case.labels_a) if len(case.labels_b) == 3
                     else (case.labels_a, case.labels_b))
    batch = third[0]                                   # unit-stride (extended) mode
    free2 = next(l for l in second if l != "k")        # the MMA N extent
    ext = {l: 200 for l in "mnp"}
    ext.update({batch: 22, free2: 256, "k": 132})
    err, kern = _strided_case_run(cid, ext, 24, dtype, seed=11, alpha=1.5, beta=-0.5)
    want_kern = "tc_tf32x3_pair_bb" if dtype == torch.float32 else "tc_dmma_f64_bb"
    assert kern.startswith(want_kern), (cid, kern)
    assert err <= TOL[dtype], (cid, err, kern)


# ------------------------------------------------------------------ HOOI eigensolver (subspace)


def test_top_eigh_matches_full_eigh_with_gap():
    """Subspace iteration + Rayleigh-Ritz on a gapped PSD Gram equals the full
    eigendecomposition's leading pairs (values and sign-fixed vectors)."""
    from paper_1606_05696_b200 import tucker as tk
    rng = np.random.default_rng(5)
    n, r = 384, 24
    x = rng.standard_normal((n, r)) @ np.diag(np.linspace(10, 3, r)) @ rng.standard_normal((r, 600))
    x += 1e-3 * rng.standard_normal((n, 600))
    g = torch.as_tensor(x @ x.T, device="cuda")
    w, v, its = tk.top_eigh(g, r)
    assert its > 0, "expected the subspace path"
    wr, vr = np.linalg.eigh(x @ x.T)
    wr, vr = wr[::-1][:r], vr[:, ::-1][:, :r]
    np.testing.assert_allclose(w.cpu().numpy(), wr, rtol=1e-11)
    vs = tk._sign_fix(v).cpu().numpy()
    vrs = tk._sign_fix(torch.as_tensor(vr.copy())).numpy()
    np.testing.assert_allclose(vs, vrs, atol=1e-9)
    # warm start from the answer converges in one sweep
    _, _, its2 = tk.top_eigh(g, r, q0=v)
    assert its2 == 1


def test_top_eigh_falls_back_without_gap():
    """No eigengap (white noise Gram): the solver must still return the exact
    leading pairs (full eigh fallback)."""
    from paper_1606_05696_b200 import tucker as tk
    rng = np.random.default_rng(6)
    n, r = 256, 32
    x = rng.standard_normal((n, n))
    g = torch.as_tensor(x @ x.T, device="cuda")
    w, v, _ = tk.top_eigh(g, r)
    wr = np.linalg.eigh(x @ x.T)[0][::-1][:r]
    np.testing.assert_allclose(w.cpu().numpy(), wr, rtol=1e-10)
    gv = (x @ x.T) @ v.cpu().numpy()
    np.testing.assert_allclose(gv, v.cpu().numpy() * w.cpu().numpy(), atol=1e-8 * wr[0])


def test_hooi_subspace_path_matches_oracle():
    """HOOI at a size that takes the subspace eigensolver (n >= 128) agrees
    with the CPU restatement (numpy eigh) on fit history and factor subspaces."""
    from oracle import tucker as otucker
    rng = np.random.default_rng(10)
    dims, ranks = (160, 144, 136), (8, 8, 6)
    core = rng.standard_normal(ranks)
    us = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
    full = np.einsum("abc,ia,jb,kc->ijk", core, *us) + 1e-3 * rng.standard_normal(dims)
    # fp32: the rank products run the unbiased narrow-tile mode (round-to-
    # nearest TF32 split, step accumulators summed in RN fp32), so the fit
    # -- which amplifies a relative bias e in |G|^2 by |G|^2 / (2 |T| resid) --
    # meets the north_star fp32 tolerance, rel 1e-5
    for dtype, frtol, utol in (("float64", 1e-10, 1e-8), ("float32", 1e-5, 1e-4)):
        t = DenseTensor.from_array(full, dtype=dtype)
        model = sbt.hooi(t, ranks, max_iters=3, tol=-1.0)
        ref = otucker.hooi(t.to_array().astype(np.float64), ranks, max_iters=3, tol=-1.0)
        np.testing.assert_allclose(model.fit_history, ref["fit_history"], rtol=frtol, atol=0)
        for r in range(3):
            u = model.factors[r].cpu().numpy()
            ur = ref["factors"][r]
            np.testing.assert_allclose(u, ur, atol=utol)


def _gapped_gram(rng, n, r, cols=600):
    x = rng.standard_normal((n, r)) @ np.diag(np.linspace(10, 3, r)) @ rng.standard_normal((r, cols))
    x += 1e-3 * rng.standard_normal((n, cols))
    return x @ x.T


@pytest.mark.parametrize("n,rank,fused", [(256, 16, 0), (512, 32, 0), (200, 13, 1), (384, 48, 1),
                                          (512, 32, 1), (1000, 64, 1)])
def test_ritz_kernel_matches_host_rayleigh_ritz(n, rank, fused):
    """sbt_ritz_f64 (device Jacobi + Ritz vectors + residual test + sign rule)
    equals the host Rayleigh-Ritz step of top_eigh on the same sweep."""
    import ctypes
    from paper_1606_05696_b200 import _lib
    rng = np.random.default_rng(n + rank)
    g = _gapped_gram(rng, n, rank + 4)
    wr, vr = np.linalg.eigh(g)
    wr, vr = wr[::-1], vr[:, ::-1]
    # warm basis: exact leading vectors, slightly perturbed, orthonormalised
    q = np.linalg.qr(vr[:, :rank] + 1e-4 * rng.standard_normal((n, rank)))[0]
    qz = np.concatenate([q.T, (g @ q).T])                 # [Q | Z] as rows
    m = qz @ (g @ q)                                      # [Q Z]^T Z, (2p, p)
    dq = torch.as_tensor(qz, device="cuda").contiguous()
    dm = torch.as_tensor(np.asfortranarray(m).ravel(order="F"), device="cuda")
    ut = torch.empty(rank, n, dtype=torch.float64, device="cuda")
    yt = torch.empty_like(ut)
    u32 = torch.empty(rank, n, dtype=torch.float32, device="cuda")
    w = torch.empty(rank, dtype=torch.float64, device="cuda")
    flag = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    rel = torch.empty(6, dtype=torch.float64, device="cuda")
    P = ctypes.c_void_p
    _lib.check(_lib.load().sbt_ritz_f64(
        P(dq.data_ptr()), P(dm.data_ptr()) if fused == 0 else None, n, rank, rank, 1e-12,
        P(ut.data_ptr()), P(yt.data_ptr()), P(u32.data_ptr()), P(w.data_ptr()),
        P(flag.data_ptr()), P(rel.data_ptr()), P(0)), "ritz")
    torch.cuda.synchronize()
    h = m[:rank]
    hw, hv = np.linalg.eigh(0.5 * (h + h.T))
    hw, hv = hw[::-1], hv[:, ::-1]
    np.testing.assert_allclose(w.cpu().numpy(), hw, rtol=1e-12)
    u = q @ hv
    u = u * np.where(u[np.argmax(np.abs(u), axis=0), np.arange(rank)] < 0, -1.0, 1.0)
    np.testing.assert_allclose(ut.cpu().numpy().T, u, atol=1e-10)
    assert torch.equal(u32, ut.to(torch.float32))
    r = np.linalg.norm(g @ u - u * hw, axis=0).max() / hw[0]
    assert abs(rel[0].item() - r) <= 1e-6 * r + 1e-15
    # nearly diagonal H: Newton refinement steps, few or no Jacobi sweeps
    assert 1 <= rel[5].item() + rel[1].item() and rel[1].item() <= 6
    assert flag.item() == int(r <= 1e-12)
    # Y = G U before the sign rule: |Y| columns match G u
    np.testing.assert_allclose(np.abs(yt.cpu().numpy().T), np.abs(g @ u), atol=1e-8 * hw[0])


@pytest.mark.parametrize("dims,mode,rank,dtype", [
    ((512, 32, 32), 0, 32, "float32"), ((32, 512, 32), 1, 32, "float32"),
    ((32, 32, 512), 2, 32, "float32"), ((200, 24, 17), 0, 13, "float64"),
    ((9, 300, 14), 1, 40, "float64"), ((6, 5, 7, 260), 3, 64, "float32"),
    ((7, 140, 3, 5), 1, 20, "float64")])
def test_hooi_factor_matches_host_sweep(dims, mode, rank, dtype):
    """sbt_hooi_factor_* (G Q = Y_(r) (Y_(r)^T Q) straight from the packed
    tensor, then the Ritz finish) equals the host sweep: Z against the fp64
    Gram of the mode-r unfolding, the Ritz values / sign-fixed vectors against
    numpy's Rayleigh-Ritz on the same basis (reference tucker.py:63-76)."""
    import ctypes
    from paper_1606_05696_b200 import _lib, tucker as tk
    rng = np.random.default_rng(sum(dims) + mode)
    # gapped mode-r spectrum: x = (U diag(s)) x_r G + noise, so the Ritz
    # vectors are well conditioned
    n = dims[mode]
    big = rank + 4
    others = [d for i, d in enumerate(dims) if i != mode]
    basis = np.linalg.qr(rng.standard_normal((n, big)))[0] * np.linspace(10, 3, big)
    x = np.moveaxis(np.tensordot(basis, rng.standard_normal([big] + others), axes=(1, 0)),
                    0, mode)
    x += 1e-3 * rng.standard_normal(dims)
    t = DenseTensor.from_array(x, dtype=dtype)
    xr = t.host_data().astype(np.float64).reshape(dims[::-1]).transpose(
        *reversed(range(len(dims))))             # the tensor's exact (rounded) values
    ymat = np.moveaxis(xr, mode, 0).reshape(n, -1)
    g = ymat @ ymat.T
    gw, gv = np.linalg.eigh(g)
    q = np.linalg.qr(gv[:, ::-1][:, :rank] + 1e-4 * rng.standard_normal((n, rank)))[0]
    warm = torch.as_tensor(q, device="cuda")
    status = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    u = tk._factor_device(t, mode, rank, warm, status, 0)
    torch.cuda.synchronize()
    # Z = G Q as the library computed it (workspace), fp64 accumulation
    ws = tk._factor_ws(t.data.device, tuple(dims), mode, rank)
    cd = (ctypes.c_int64 * len(dims))(*dims)
    lib = _lib.load()
    nbytes = lib.sbt_hooi_factor_ws_bytes(len(dims), cd, mode, rank)
    assert nbytes == ws.numel()
    z_want = g @ q
    h = q.T @ z_want
    hw, hv = np.linalg.eigh(0.5 * (h + h.T))
    hw, hv = hw[::-1], hv[:, ::-1]
    uw = q @ hv
    uw = uw * np.where(uw[np.argmax(np.abs(uw), axis=0), np.arange(rank)] < 0, -1.0, 1.0)
    # the Ritz kernel stops rotating at off-diagonals <= 1e-2 tol ||H|| (tol =
    # 1e-12 fp64, 1e-6 fp32 tensors: their data carry ~1e-7 relative error)
    np.testing.assert_allclose(u.cpu().numpy(), uw, atol=1e-9 if dtype == "float64" else 5e-6)
    assert status.item() in (0, 1)
    # Z = G Q as the library left it in the workspace (after W: cols x p)
    cols = int(np.prod(dims)) // n
    z = ws.view(torch.float64)[cols * rank:cols * rank + rank * n].reshape(rank, n).t()
    np.testing.assert_allclose(z.cpu().numpy(), z_want, rtol=0,
                               atol=1e-12 * np.abs(z_want).max())


@pytest.mark.parametrize("dims,mode,rank,dtype", [
    ((32, 32, 512), 2, 32, "float32"), ((17, 40, 23), 1, 7, "float32"),
    ((64, 9, 5, 6), 0, 64, "float64"), ((5, 6, 7, 33), 3, 3, "float32")])
def test_mode_product_acc64_matches_oracle(dims, mode, rank, dtype):
    """sbt_mode_product_acc64_* (the HOOI core product with fp64 accumulation)
    equals the fp64 mode product of the same values, rounded once."""
    from paper_1606_05696_b200 import tucker as tk
    rng = np.random.default_rng(sum(dims) * 3 + mode)
    x = rng.uniform(-1, 1, dims)
    t = DenseTensor.from_array(x, dtype=dtype)
    xr = t.to_array().astype(np.float64)
    u = rng.standard_normal((dims[mode], rank))
    got = tk._mode_product_acc64(t, torch.as_tensor(u, device="cuda"), mode)
    want = np.moveaxis(np.tensordot(xr, u, axes=([mode], [0])), -1, mode)
    assert got.layout == Layout.packed(want.shape)
    rtol = 1e-13 if dtype == "float64" else 6e-8
    np.testing.assert_allclose(got.to_array().astype(np.float64), want,
                               rtol=rtol, atol=rtol * np.abs(want).max())


def test_hooi_sharded_device_ops_single_rank_equals_hooi():
    """parallel.hooi_sharded on the device path (DeviceOps: planned mode
    products, ring Gram, device-finished factor updates, status kernel) with
    one NCCL rank gives hooi()'s fits and factors."""
    import torch.distributed as dist
    from paper_1606_05696_b200.parallel import hooi_sharded
    rng = np.random.default_rng(31)
    dims, ranks = (256, 192, 160), (16, 12, 8)
    core = rng.standard_normal(ranks)
    us = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
    full = np.einsum("abc,ia,jb,kc->ijk", core, *us) + 1e-3 * rng.standard_normal(dims)
    dist.init_process_group("nccl", rank=0, world_size=1, store=dist.HashStore(),
                            device_id=torch.device("cuda", 0))
    try:
        for dtype, ftol, utol in (("float64", 1e-12, 1e-9), ("float32", 1e-6, 1e-5)):
            t = DenseTensor.from_array(full, dtype=dtype)
            m = sbt.hooi(t, ranks, max_iters=4, tol=-1.0, use_graph=False)
            _, u, fits, iters = hooi_sharded(t, dims, ranks, max_iters=4, tol=-1.0)
            assert iters == 4
            np.testing.assert_allclose(fits, m.fit_history, rtol=0, atol=ftol)
            for u1, u2 in zip(u, m.factors):
                np.testing.assert_allclose(u1.cpu().numpy(), u2.cpu().numpy(), atol=utol)
    finally:
        dist.destroy_process_group()


def test_hooi_iteration_graph_runs_only_library_kernels():
    """The captured HOOI iteration (device-finished factor updates) launches
    library kernels only: no PyTorch elementwise / reduction / copy kernels
    between the contractions, the factor updates and the status kernel."""
    from torch.profiler import ProfilerActivity, profile
    from paper_1606_05696_b200 import tucker as tk
    rng = np.random.default_rng(41)
    dims, ranks = (160, 144, 128), (8, 8, 8)
    core = rng.standard_normal(ranks)
    us = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
    full = np.einsum("abc,ia,jb,kc->ijk", core, *us) + 1e-3 * rng.standard_normal(dims)
    t = DenseTensor.from_array(full, dtype="float32")
    tk.clear_graph_cache()
    sbt.hooi(t, ranks, max_iters=5, tol=-1.0)
    cached = tk._IterationGraph._cache
    assert cached is not None, "the iteration graph was not captured"
    graph = cached[1]
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        graph.graphs[graph.cur].replay()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events()
             if e.device_type == torch.autograd.DeviceType.CUDA and "Memcpy" not in e.name
             and "Memset" not in e.name]
    assert names, "no kernels recorded"
    foreign = [n for n in names if "sbt::" not in n]
    assert not foreign, foreign
    tk.clear_graph_cache()


def test_hooi_device_ritz_equals_host_path():
    """HOOI with the device-finished sweeps (one host sync per iteration)
    gives the host-driven path's fits and factors, fp32 and fp64."""
    rng = np.random.default_rng(21)
    dims, ranks = (256, 192, 160), (16, 12, 8)
    core = rng.standard_normal(ranks)
    us = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
    full = np.einsum("abc,ia,jb,kc->ijk", core, *us) + 1e-3 * rng.standard_normal(dims)
    for dtype, ftol, utol in (("float64", 1e-12, 1e-9), ("float32", 1e-6, 1e-5)):
        t = DenseTensor.from_array(full, dtype=dtype)
        m1 = sbt.hooi(t, ranks, max_iters=4, tol=-1.0, device_ritz=True)
        m2 = sbt.hooi(t, ranks, max_iters=4, tol=-1.0, device_ritz=False)
        np.testing.assert_allclose(m1.fit_history, m2.fit_history, rtol=0, atol=ftol)
        for u1, u2 in zip(m1.factors, m2.factors):
            np.testing.assert_allclose(u1.cpu().numpy(), u2.cpu().numpy(), atol=utol)


def test_hooi_graph_replay_equals_eager():
    """The CUDA-graph replay of the device-finished iteration gives bitwise
    the eager iteration's fits and factors (same kernels, same order)."""
    rng = np.random.default_rng(22)
    dims, ranks = (256, 160, 192), (16, 8, 12)
    core = rng.standard_normal(ranks)
    us = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
    full = np.einsum("abc,ia,jb,kc->ijk", core, *us) + 1e-3 * rng.standard_normal(dims)
    for dtype in ("float32", "float64"):
        t = DenseTensor.from_array(full, dtype=dtype)
        m1 = sbt.hooi(t, ranks, max_iters=6, tol=-1.0, use_graph=True)
        m2 = sbt.hooi(t, ranks, max_iters=6, tol=-1.0, use_graph=False)
        assert m1.fit_history == m2.fit_history
        for u1, u2 in zip(m1.factors, m2.factors):
            assert torch.equal(u1, u2)


def test_device_ritz_flags_unconverged_sweep():
    """A poor warm start does not converge in one sweep: the flag is 0 (HOOI
    then recomputes the iteration on the host path)."""
    from paper_1606_05696_b200 import tucker as tk
    rng = np.random.default_rng(3)
    n, rank = 256, 16
    x = rng.standard_normal((n, 4000))
    t = DenseTensor.from_array(x.reshape(n, 40, 100), dtype="float64")
    warm = torch.linalg.qr(torch.randn(n, rank, dtype=torch.float64, device="cuda"))[0]
    status = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    u = tk._factor_device(t, 0, rank, warm, status, 0)
    torch.cuda.synchronize()
    assert status.item() == 0
    assert u.shape == (n, rank)


@pytest.mark.parametrize("m,n,k,P", [(256, 256, 8192, 2), (128, 128, 40000, 1), (512, 320, 3000, 3)])
def test_fp32_long_reductions_stay_within_tolerance(m, n, k, P):
    """3xTF32 truncation bias grows with K; long reductions are K-chunked (and
    split-K partials too) so max_rel_err stays <= 1e-5 at any K."""
    rng = np.random.default_rng(k)
    ha, hb = rng.uniform(-1, 1, m * k * P), rng.uniform(-1, 1, k * n * P)
    a, b = dev(ha, torch.float32), dev(hb, torch.float32)
    c = torch.zeros(m * n * P, dtype=torch.float32, device="cuda")
    kernels.strided_batched_gemm("N", "N", m, n, k, 1.0, a, m, m * k, b, k, k * n, 0.0, c, m,
                                 m * n, P)
    A = host(a).reshape(P, k, m).transpose(0, 2, 1)
    B = host(b).reshape(P, n, k).transpose(0, 2, 1)
    want = np.einsum("pik,pkj->pij", A, B)
    got = host(c).reshape(P, n, m).transpose(0, 2, 1)
    assert naive.max_rel_err(got, want) <= TOL[torch.float32]


# ------------------------------------------------------------------ batch folding (pair kernel)


def test_fourth_order_n128_folds_both_batch_modes():
    """C[mnpq] = A[mkp] B[nkq] at n=128 (BASELINE configs[4]): one launch of
    the CTA-pair kernel with p folded into M and q into N; sampled (p, q)
    slices against fp64 matmuls."""
    n = 128
    rng = np.random.default_rng(44)
    spec = ContractionSpec(tuple("mkp"), tuple("nkq"), tuple("mnpq"))
    la, lb, lc = Layout.packed((n,) * 3), Layout.packed((n,) * 3), Layout.packed((n,) * 4)
    ha, hb = rng.uniform(-1, 1, la.size), rng.uniform(-1, 1, lb.size)
    a = DenseTensor(la, dev(ha, torch.float32))
    b = DenseTensor(lb, dev(hb, torch.float32))
    c = DenseTensor(lc, torch.full((lc.size,), float("nan"), dtype=torch.float32, device="cuda"))
    n0 = _lib.launch_count()
    execute_plan(plan_single_mode(spec, la, lb, lc), a, b, 1.0, 0.0, c)
    torch.cuda.synchronize()
    assert _lib.launch_count() - n0 == 1
    assert _lib.last_kernel().startswith("tc_tf32x3_pair_fold"), _lib.last_kernel()
    A = host(a.data).reshape(n, n, n)     # [p][k][m]
    B = host(b.data).reshape(n, n, n)     # [q][k][n]
    C = c.data.view(n, n, n, n)           # [q][p][n][m]
    for (p, q) in [(0, 0), (127, 127), (5, 77), (64, 3), (100, 126)] + \
            [tuple(x) for x in rng.integers(0, n, (8, 2))]:
        want = (A[p].T @ B[q])            # [m][n]
        got = C[q, p].double().cpu().numpy().T
        assert naive.max_rel_err(got, want) <= TOL[torch.float32], (p, q)
    assert not torch.isnan(C).any()


@pytest.mark.parametrize("shape", [
    # m, n, k, batch, aps, bps : fold batch into M (B broadcast) / into N (A broadcast)
    (384, 256, 96, 5, "a", 0),
    (256, 384, 200, 3, 0, "b"),
    (640, 256, 64, 4, "a", 0),
    # fewer than 128 rows per batch entry (MN-major A: 32-row boxes per entry)
    (32, 32, 512, 512, "a", 0),
    (96, 32, 200, 200, "a", 0),
    (160, 64, 72, 64, "a", 0),
])
def test_batch_fold_into_m_or_n(shape):
    m, n, k, P, aps, bps = shape
    rng = np.random.default_rng(m + n + k)
    aps = m * k if aps == "a" else 0
    bps = k * n if bps == "b" else 0
    ha = rng.uniform(-1, 1, m * k * (P if aps else 1))
    hb = rng.uniform(-1, 1, k * n * (P if bps else 1))
    hc = rng.uniform(-1, 1, m * n * P)
    a, b, c = dev(ha, torch.float32), dev(hb, torch.float32), dev(hc, torch.float32)
    kernels.strided_batched_gemm("N", "N", m, n, k, 1.5, a, m, aps, b, k, bps, -0.25, c, m,
                                 m * n, P)
    kern = _lib.last_kernel()
    want = host(dev(hc, torch.float32)).copy()
    oapi.run_call("strided_batched_gemm", dict(opa="N", opb="N", m=m, n=n, k=k, alpha=1.5,
                  lda=m, loa=aps, ldb=k, lob=bps, beta=-0.25, ldc=m, loc=m * n, batch_count=P),
                  host(a), host(b), want)
    assert kern.startswith("tc_tf32x3_pair_fold"), kern
    assert naive.max_rel_err(host(c), want) <= TOL[torch.float32]


@pytest.mark.parametrize("m,n,k,P", [(16384, 32, 256, 1), (8192, 48, 100, 1), (12000, 20, 64, 1),
                                     (512, 32, 512, 40)])
def test_narrow_tiles_for_skinny_products(m, n, k, P):
    """Rank-r style products (long M', N <= 64, K-major B) run on the CTA-pair
    kernel with 32/64-wide tiles (batch folded into M when B is shared)."""
    rng = np.random.default_rng(m + n)
    ha = rng.uniform(-1, 1, m * k * P)
    hb = rng.uniform(-1, 1, k * n)
    a, b = dev(ha, torch.float32), dev(hb, torch.float32)
    c = torch.zeros(m * n * P, dtype=torch.float32, device="cuda")
    kernels.strided_batched_gemm("N", "N", m, n, k, 1.0, a, m, m * k, b, k, 0, 0.0, c, m, m * n,
                                 P)
    assert _lib.last_kernel().startswith("tc_tf32x3_pair"), _lib.last_kernel()
    A = host(a).reshape(P, k, m).transpose(0, 2, 1)
    B = host(b).reshape(n, k).T
    want = A @ B
    got = host(c).reshape(P, n, m).transpose(0, 2, 1)
    assert naive.max_rel_err(got, want) <= TOL[torch.float32]


# ------------------------------------------------------------------ grouped execution


@pytest.mark.parametrize("n,dtype", [(64, torch.float32), (128, torch.float32),
                                     (256, torch.float32), (64, torch.float64)])
def test_grouped_execution_equals_single_calls(n, dtype):
    """execute_plans (one persistent launch per kernel configuration) gives
    bitwise the results of per-call execute_plan for all 36 cases, with
    distinct outputs, and matches the oracle."""
    rng = np.random.default_rng(n)
    calls, singles = [], []
    for i, case in enumerate(enumerate_cases(2, 3)):
        spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
        la, lb, lc = _packed(spec, dict(m=n, n=n, p=n, k=n))
        a = DenseTensor(la, dev(rng.uniform(-1, 1, la.size), dtype))
        b = DenseTensor(lb, dev(rng.uniform(-1, 1, lb.size), dtype))
        c0 = rng.uniform(-1, 1, lc.size)
        beta = 0.5 if i % 5 == 0 else 0.0
        plan = plan_single_mode(spec, la, lb, lc)
        cg = DenseTensor(lc, dev(c0, dtype))
        cs = DenseTensor(lc, dev(c0, dtype))
        calls.append((plan, a, b, 1.25, beta, cg))
        singles.append((plan, a, b, 1.25, beta, cs))
    n0 = _lib.launch_count()
    sbt.execute_plans(calls)
    torch.cuda.synchronize()
    grouped_launches = _lib.launch_count() - n0
    for plan, a, b, al, be, cs in singles:
        execute_plan(plan, a, b, al, be, cs)
    torch.cuda.synchronize()
    if dtype == torch.float32 and n >= 128:
        assert grouped_launches < 36, grouped_launches
    for (plan, a, b, al, be, cg), (_, _, _, _, _, cs) in zip(calls, singles):
        assert torch.equal(cg.data, cs.data), plan.spec
    # and one of them (beta = 0) against the oracle
    plan, a, b, al, be, cg = calls[-2]
    assert be == 0.0
    spec = plan.spec
    ext = dict(m=n, n=n, p=n, k=n)
    want = np.zeros(plan.layout_c.size)
    oplan.contract(spec.labels_a, spec.labels_b, spec.labels_c, ext, host(a.data),
                   host(b.data), al, 0.0, want)
    assert naive.max_rel_err(host(cg.data), want) <= TOL[dtype]


def test_grouped_execution_rejects_dependent_calls():
    spec = ContractionSpec(tuple("mk"), tuple("knp"), tuple("mnp"))
    la, lb, lc = Layout.packed((8, 4)), Layout.packed((4, 8, 8)), Layout.packed((8, 8, 8))
    a = DenseTensor(la, dev(np.ones(la.size)))
    b = DenseTensor(lb, dev(np.ones(lb.size)))
    c = DenseTensor(lc, dev(np.zeros(lc.size)))
    plan = plan_single_mode(spec, la, lb, lc)
    with pytest.raises(ValueError):
        sbt.execute_plans([(plan, a, b, 1.0, 0.0, c), (plan, a, b, 1.0, 0.0, c)])


@pytest.mark.parametrize("P,beta,mma", [(2001, 0.0, 1), (999, 0.5, 1), (2001, 0.0, 0),
                                        (999, 0.5, 0)])
def test_small64_fp32(P, beta, mma, monkeypatch):
    """fp32 64^3 batches: the mma.sync 3xTF32 kernel (default) or, with
    SBT_SMALL64_MMA=0 in the environment (read once by the library), the
    8x8-register-blocked FFMA kernel -- odd batch, beta != 0."""
    n = 64
    import os
    if mma != (os.environ.get("SBT_SMALL64_MMA", "1") != "0"):
        pytest.skip("variant selected by SBT_SMALL64_MMA (tools/check_small64.sh runs both)")
    rng = np.random.default_rng(P)
    ha, hb, hc = (rng.uniform(-1, 1, n * n * P) for _ in range(3))
    a, b, c = dev(ha, torch.float32), dev(hb, torch.float32), dev(hc, torch.float32)
    kernels.strided_batched_gemm("N", "N", n, n, n, 1.5, a, n, n * n, b, n, n * n, beta, c, n,
                                 n * n, P)
    assert _lib.last_kernel() == ("small64_mma_f32" if mma else "small64_f32")
    A = host(a).reshape(P, n, n).transpose(0, 2, 1)
    B = host(b).reshape(P, n, n).transpose(0, 2, 1)
    want = (1.5 * (A @ B)).transpose(0, 2, 1).reshape(-1) + beta * host(dev(hc, torch.float32))
    assert naive.max_rel_err(host(c), want) <= TOL[torch.float32]


@pytest.mark.parametrize("m,n,k,opa,opb", [(1024, 32, 512, "T", "N"), (512, 32, 1024, "N", "N"),
                                           (64, 32, 512, "T", "N"), (200, 40, 333, "N", "T"),
                                           (48, 700, 96, "T", "T"), (16384, 32, 512, "N", "N")])
def test_skinny_fp64_products(m, n, k, opa, opb):
    """fp64 products with a narrow side (the HOOI rank-p products) run on the
    skinny DMMA kernel (in-kernel split-K, fixed reduction order): parity with
    the oracle at 1e-12 and bitwise-reproducible."""
    rng = np.random.default_rng(m * 7 + n + k)
    lda = m if opa == "N" else k
    ldb = k if opb == "N" else n
    ha = rng.uniform(-1, 1, m * k)
    hb = rng.uniform(-1, 1, k * n)
    hc = rng.uniform(-1, 1, m * n)
    a, b = dev(ha, torch.float64), dev(hb, torch.float64)
    outs = []
    for _ in range(2):
        c = dev(hc, torch.float64)
        kernels.gemm(opa, opb, m, n, k, 0.75, a, lda, b, ldb, 0.5, c, m)
        outs.append(c)
    assert _lib.last_kernel() == "skinny_dmma_f64", _lib.last_kernel()
    assert torch.equal(outs[0], outs[1])
    # column-major buffers: A is m x k (N, ld m) or stored k x m (T, ld k)
    A = ha.reshape(k, m).T if opa == "N" else ha.reshape(m, k)
    B = hb.reshape(n, k).T if opb == "N" else hb.reshape(k, n)
    want = 0.75 * A @ B + 0.5 * hc.reshape(n, m).T
    got = host(outs[0]).reshape(n, m).T
    assert naive.max_rel_err(got, want) <= TOL[torch.float64]


@pytest.mark.parametrize("m,n,k,P,bcast", [(512, 32, 512, 6, True), (96, 40, 200, 5, False),
                                           (64, 64, 64, 7, False)])
def test_skinny_fp64_batched(m, n, k, P, bcast):
    """Batched fp64 products with a <= 64-wide side (fp64 Tucker mode products)
    run on the skinny kernel, one grid slice per batch entry."""
    rng = np.random.default_rng(m + n + k + P)
    ha = rng.uniform(-1, 1, m * k * P)
    hb = rng.uniform(-1, 1, k * n * (1 if bcast else P))
    hc = rng.uniform(-1, 1, m * n * P)
    a, b, c = dev(ha, torch.float64), dev(hb, torch.float64), dev(hc, torch.float64)
    lob = 0 if bcast else k * n
    kernels.strided_batched_gemm("N", "N", m, n, k, 1.25, a, m, m * k, b, k, lob, -0.5, c, m,
                                 m * n, P)
    assert _lib.last_kernel() == "skinny_dmma_f64", _lib.last_kernel()
    want = host(dev(hc, torch.float64)).copy()
    oapi.run_call("strided_batched_gemm", dict(opa="N", opb="N", m=m, n=n, k=k, alpha=1.25,
                  lda=m, loa=m * k, ldb=k, lob=lob, beta=-0.5, ldc=m, loc=m * n, batch_count=P),
                  host(a), host(b), want)
    assert naive.max_rel_err(host(c), want) <= TOL[torch.float64]


def test_hooi_graph_cache_reused_across_calls():
    """A second hooi() on the same tensor replays the cached iteration graph
    (no recapture) and reproduces the first call bitwise."""
    from paper_1606_05696_b200 import tucker as tk
    rng = np.random.default_rng(23)
    dims, ranks = (192, 160, 128), (12, 8, 8)
    core = rng.standard_normal(ranks)
    us = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
    full = np.einsum("abc,ia,jb,kc->ijk", core, *us) + 1e-3 * rng.standard_normal(dims)
    t = DenseTensor.from_array(full, dtype="float32")
    tk.clear_graph_cache()
    m1 = sbt.hooi(t, ranks, max_iters=6, tol=-1.0)
    g1 = tk._IterationGraph._cache[1]
    m2 = sbt.hooi(t, ranks, max_iters=6, tol=-1.0)
    assert tk._IterationGraph._cache[1] is g1
    assert m1.stats["graph"] and m2.stats["device_iterations"] >= 5
    assert m1.fit_history == m2.fit_history
    for u1, u2 in zip(m1.factors, m2.factors):
        assert torch.equal(u1, u2)
    tk.clear_graph_cache()
    assert tk._IterationGraph._cache is None


@pytest.mark.parametrize("m,n,k", [(64, 64, 64), (48, 40, 64), (64, 24, 36), (40, 64, 20)])
def test_small_dmma64_fp64(m, n, k):
    """fp64 batches of matrices with an extent in (32, 64] run on the DMMA
    small-matrix kernel (four warps per matrix) and match the oracle."""
    P = 700
    rng = np.random.default_rng(m * n + k)
    ha, hb, hc = (rng.uniform(-1, 1, m * k * P), rng.uniform(-1, 1, k * n * P),
                  rng.uniform(-1, 1, m * n * P))
    a, b, c = dev(ha, torch.float64), dev(hb, torch.float64), dev(hc, torch.float64)
    kernels.strided_batched_gemm("N", "N", m, n, k, 0.5, a, m, m * k, b, k, k * n, 2.0, c, m,
                                 m * n, P)
    assert _lib.last_kernel() == "small_batched_dmma64_f64", _lib.last_kernel()
    want = host(dev(hc, torch.float64)).copy()
    oapi.run_call("strided_batched_gemm", dict(opa="N", opb="N", m=m, n=n, k=k, alpha=0.5,
                  lda=m, loa=m * k, ldb=k, lob=k * n, beta=2.0, ldc=m, loc=m * n, batch_count=P),
                  host(a), host(b), want)
    assert naive.max_rel_err(host(c), want) <= TOL[torch.float64]


@pytest.mark.parametrize("m,n,k,P,ldc_pad", [(1000, 300, 96, 3, 0), (1000, 300, 96, 3, 8),
                                             (4100, 256, 64, 1, 4), (520, 1030, 40, 2, 0)])
def test_tma_store_epilogue_clips_tails(m, n, k, P, ldc_pad):
    """beta = 0 pair-kernel calls use the per-warp TMA-store epilogue: row /
    column tails that are not multiples of the 32 x 32 store box are clipped by
    the tensor map, padded leading dimensions are respected (padding untouched)."""
    rng = np.random.default_rng(m + n + ldc_pad)
    ldc = m + ldc_pad
    ha, hb = rng.uniform(-1, 1, m * k * P), rng.uniform(-1, 1, k * n * P)
    a, b = dev(ha, torch.float32), dev(hb, torch.float32)
    sentinel = 7.0
    c = torch.full((ldc * n * P,), sentinel, dtype=torch.float32, device="cuda")
    kernels.strided_batched_gemm("N", "N", m, n, k, 1.0, a, m, m * k, b, k, k * n, 0.0, c, ldc,
                                 ldc * n, P)
    assert _lib.last_kernel().startswith("tc_tf32x3_pair"), _lib.last_kernel()
    A = ha.reshape(P, k, m).transpose(0, 2, 1)
    B = hb.reshape(P, n, k).transpose(0, 2, 1)
    want = np.einsum("pik,pkj->pij", A, B)
    full = host(c).reshape(P, n, ldc).transpose(0, 2, 1)
    assert naive.max_rel_err(full[:, :m, :], want) <= TOL[torch.float32]
    if ldc_pad:
        assert np.all(full[:, m:, :] == sentinel)
