"""Parity at the BASELINE configurations (BASELINE.json configs[0..4]) against
the CPU oracle, at the sizes the bench runs:

* every one of the 36 single-index cases at n = 256 and n = 512, fp32 and fp64
  (configs[1]); the inputs are fp32-representable so one fp64 oracle run
  serves both dtypes (fp32 = fp64 oracle on the same fp32 values, SURVEY.md
  section 8c);
* n = 1024 on sampled output entries (each sampled entry's k-sum computed in
  fp64 on the host from the operands);
* the exact configs[0] call, device buffers and host (numpy) buffers;
* Tucker HOOI 512^3 rank 32 fp32 (configs[3]): fit history within rel 1e-5 of
  the fp64 oracle (oracle/tucker.py, reference tucker.py:136-174) run on the
  same fp32 tensor, and the factor subspaces.

Tolerances (north_star): max_rel_err <= 1e-12 fp64, <= 1e-5 fp32.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1606_05696_b200 as sbt  # noqa: E402
from paper_1606_05696_b200 import kernels  # noqa: E402
from paper_1606_05696_b200.layout import DenseTensor, Layout  # noqa: E402
from paper_1606_05696_b200.notation import ContractionSpec  # noqa: E402
from paper_1606_05696_b200.planner import enumerate_cases, execute_plan, plan_single_mode  # noqa
from oracle import cores as ocores, naive, plan as oplan  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = {torch.float64: 1e-12, torch.float32: 1e-5}
CASES = [c.case_id for c in enumerate_cases(2, 3)]


def _spec_layouts(cid, n):
    case = sbt.find_case(2, 3, cid)
    spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
    ext = dict(m=n, n=n, p=n, k=n)
    lays = tuple(Layout.packed([ext[l] for l in labs])
                 for labs in (spec.labels_a, spec.labels_b, spec.labels_c))
    return spec, ext, lays


def _f32_values(rng, size):
    """U[-1,1] rounded to fp32 (exact in both dtypes)."""
    return rng.uniform(-1, 1, size).astype(np.float32).astype(np.float64)


def _device_run(spec, lays, ha, hb, dtype, alpha=1.0, beta=0.0, hc=None):
    a = DenseTensor(lays[0], torch.from_numpy(ha).to("cuda", dtype))
    b = DenseTensor(lays[1], torch.from_numpy(hb).to("cuda", dtype))
    c = (DenseTensor(lays[2], torch.from_numpy(hc).to("cuda", dtype)) if hc is not None
         else DenseTensor.zeros(lays[2], dtype=dtype))
    execute_plan(plan_single_mode(spec, *lays), a, b, alpha, beta, c)
    out = c.data.double().cpu().numpy()
    del a, b, c
    return out


@pytest.mark.parametrize("n", [256, 512])
@pytest.mark.parametrize("cid", CASES)
def test_all_36_cases_large_vs_oracle(cid, n):
    """Every case at the sweep extents, both dtypes against one fp64 oracle
    run; every third case with beta != 0 (C read and scaled)."""
    spec, ext, lays = _spec_layouts(cid, n)
    rng = np.random.default_rng(CASES.index(cid) * 7919 + n)
    ha, hb = _f32_values(rng, lays[0].size), _f32_values(rng, lays[1].size)
    beta = 0.5 if CASES.index(cid) % 3 == 0 else 0.0
    alpha = 1.25
    hc = _f32_values(rng, lays[2].size) if beta else None
    want = hc.copy() if beta else np.zeros(lays[2].size)
    oplan.contract(spec.labels_a, spec.labels_b, spec.labels_c, ext, ha, hb, alpha, beta, want)
    for dtype in (torch.float64, torch.float32):
        got = _device_run(spec, lays, ha, hb, dtype, alpha, beta, hc)
        err = naive.max_rel_err(got, want)
        assert err <= TOL[dtype], (cid, n, dtype, err)
    torch.cuda.empty_cache()


def _sampled_reference(spec, ext, ha, hb, rng, count):
    """fp64 values of `count` random output entries: for each sampled free
    index, the k-sum over the operands' packed column-major buffers."""
    def strides(labels):
        s, acc = {}, 1
        for l in labels:
            s[l] = acc
            acc *= ext[l]
        return s
    sa, sb, sc = strides(spec.labels_a), strides(spec.labels_b), strides(spec.labels_c)
    (klab,) = [l for l in spec.labels_a if l in spec.labels_b]
    idx = {l: rng.integers(0, ext[l], count) for l in spec.labels_c}
    ks = np.arange(ext[klab])
    oa = sum(idx[l] * sa[l] for l in spec.labels_a if l != klab)
    ob = sum(idx[l] * sb[l] for l in spec.labels_b if l != klab)
    oc = sum(idx[l] * sc[l] for l in spec.labels_c)
    va = ha[oa[:, None] + ks[None, :] * sa[klab]]
    vb = hb[ob[:, None] + ks[None, :] * sb[klab]]
    return oc, np.einsum("ij,ij->i", va, vb)


@pytest.mark.parametrize("cid", ["1.1", "1.3", "2.4", "3.6", "5.5", "6.4"])
def test_sampled_entries_n1024(cid):
    """n = 1024 (B and C hold 2^30 elements): 4096 sampled entries per case
    against fp64 k-sums on the host; max |err| / max |want| over the sample."""
    n = 1024
    spec, ext, lays = _spec_layouts(cid, n)
    rng = np.random.default_rng(CASES.index(cid) + 17)
    g = torch.Generator(device="cuda").manual_seed(CASES.index(cid))
    for dtype in (torch.float32, torch.float64):
        a = DenseTensor(lays[0], (torch.rand(lays[0].size, generator=g, device="cuda",
                                             dtype=torch.float32) * 2 - 1).to(dtype))
        b = DenseTensor(lays[1], (torch.rand(lays[1].size, generator=g, device="cuda",
                                             dtype=torch.float32) * 2 - 1).to(dtype))
        c = DenseTensor.empty(lays[2], dtype=dtype)
        execute_plan(plan_single_mode(spec, *lays), a, b, 1.0, 0.0, c)
        ha, hb = a.data.double().cpu().numpy(), b.data.double().cpu().numpy()
        oc, want = _sampled_reference(spec, ext, ha, hb, rng, 4096)
        got = c.data[torch.from_numpy(oc).cuda()].double().cpu().numpy()
        err = np.abs(got - want).max() / np.abs(want).max()
        assert err <= TOL[dtype], (cid, dtype, err)
        del a, b, c
        torch.cuda.empty_cache()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_c1_exact_call(dtype):
    """configs[0] verbatim: strided_batched_gemm('N','N',256,256,256,1,A,256,0,
    B,256,65536,0,C,256,65536,256) -- device buffers, then numpy host buffers
    through the host seam (the reference's own buffer type)."""
    n = 256
    rng = np.random.default_rng(256)
    ha, hb = _f32_values(rng, n * n), _f32_values(rng, n ** 3)
    want = np.zeros(n ** 3)
    ocores.batched_core(n, n, n, 1.0, ha, 0, 1, n, 0, hb, 0, 1, n, n * n, 0.0, want, 0, 1, n,
                        n * n, n)
    a = torch.from_numpy(ha).to("cuda", dtype)
    b = torch.from_numpy(hb).to("cuda", dtype)
    c = torch.full((n ** 3,), float("nan"), device="cuda", dtype=dtype)  # beta = 0: never read
    kernels.strided_batched_gemm("N", "N", 256, 256, 256, 1.0, a, 256, 0, b, 256, 65536, 0.0, c,
                                 256, 65536, 256)
    assert naive.max_rel_err(c.double().cpu().numpy(), want) <= TOL[dtype]
    npdt = np.float64 if dtype == torch.float64 else np.float32
    hc = np.full(n ** 3, np.nan, dtype=npdt)
    kernels.strided_batched_gemm("N", "N", 256, 256, 256, 1.0, ha.astype(npdt), 256, 0,
                                 hb.astype(npdt), 256, 65536, 0.0, hc, 256, 65536, 256)
    assert naive.max_rel_err(hc.astype(np.float64), want) <= TOL[dtype]


def _synthetic_tucker(n, r, seed=0, noise=1e-3):
    """Exact-rank Tucker tensor plus noise, fp32."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    core = torch.randn(r, r, r, device="cuda", generator=g, dtype=torch.float64)
    us = [torch.linalg.qr(torch.randn(n, r, device="cuda", generator=g,
                                      dtype=torch.float64))[0] for _ in range(3)]
    x = torch.einsum("ia,abc->ibc", us[0], core)
    x = torch.einsum("jb,ibc->ijc", us[1], x)
    x = torch.einsum("kc,ijc->ijk", us[2], x)
    x = x + noise * torch.randn(n, n, n, device="cuda", generator=g, dtype=torch.float64)
    return x.permute(2, 1, 0).contiguous().reshape(-1).to(torch.float32)


def test_hooi_c4_fp32_matches_fp64_oracle():
    """configs[3]: HOOI 512^3 rank 32 on an fp32 tensor vs the fp64 CPU
    restatement on the same values: fit history within rel 1e-5 (the
    north_star fp32 tolerance; no relaxed bound), factor subspaces within
    1e-5 (projector entries)."""
    from oracle import tucker as otucker
    n, r, iters = 512, 32, 3
    flat = _synthetic_tucker(n, r)
    t = DenseTensor(Layout.packed((n, n, n)), flat)
    model = sbt.hooi(t, (r, r, r), max_iters=iters, tol=-1.0)
    x = flat.cpu().numpy().astype(np.float64).reshape((n, n, n), order="F")
    del flat
    ref = otucker.hooi(x, (r, r, r), max_iters=iters, tol=-1.0)
    np.testing.assert_allclose(model.fit_history, ref["fit_history"], rtol=1e-5, atol=0)
    for k in range(3):
        u = model.factors[k].cpu().numpy()
        ur = ref["factors"][k]
        np.testing.assert_allclose(u @ u.T, ur @ ur.T, atol=1e-5)
    from paper_1606_05696_b200 import tucker as tk
    tk.clear_graph_cache()
