"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 paths:
slab sharding of contractions (no collective) and the sharded HOOI's
all-reduce / all-gather logic."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1606_05696_b200.layout import Layout
from paper_1606_05696_b200.notation import ContractionSpec
from paper_1606_05696_b200.parallel import (HostOps, hooi_sharded, shard_contraction,
                                            slab)
from paper_1606_05696_b200.planner import enumerate_cases


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, fn, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    errs = [o for o in out if isinstance(o, str)]
    assert not errs, errs
    return sorted(out, key=lambda o: o[0])


def _worker(rank, world, port, fn, args, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        q.put((rank, fn(rank, world, *args)))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_slab_partition():
    for n in (1, 5, 8, 13, 512):
        for w in (1, 2, 3, 8):
            parts = [slab(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


def test_shard_contraction_slabs_tile_the_output():
    """Every (2,3) case: the ranks' slab contractions reassemble the full result."""
    rng = np.random.default_rng(0)
    ext = dict(m=4, n=5, p=7, k=3)
    for case in enumerate_cases(2, 3):
        spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
        la, lb, lc = (Layout.packed([ext[l] for l in labs])
                      for labs in (spec.labels_a, spec.labels_b, spec.labels_c))
        A = rng.standard_normal(la.dims)
        B = rng.standard_normal(lb.dims)
        full = np.einsum(f"{''.join(spec.labels_a)},{''.join(spec.labels_b)}->"
                         f"{''.join(spec.labels_c)}", A, B)
        flat_a, flat_b = A.ravel(order="F"), B.ravel(order="F")
        got = np.zeros(lc.size)
        for r in range(3):
            sh = shard_contraction(spec, la, lb, lc, 3, r)
            sla, slb, slc = sh.layouts
            va = np.lib.stride_tricks.as_strided(flat_a[sh.offsets[0]:], sla.dims,
                                                 [s * 8 for s in sla.strides])
            vb = np.lib.stride_tricks.as_strided(flat_b[sh.offsets[1]:], slb.dims,
                                                 [s * 8 for s in slb.strides])
            part = np.einsum(f"{''.join(spec.labels_a)},{''.join(spec.labels_b)}->"
                             f"{''.join(spec.labels_c)}", va, vb)
            vc = np.lib.stride_tricks.as_strided(got[sh.offsets[2]:], slc.dims,
                                                 [s * 8 for s in slc.strides], writeable=True)
            vc[...] = part
        np.testing.assert_allclose(got.reshape(lc.dims, order="F"), full, atol=1e-12,
                                   err_msg=case.case_id)


def _hooi_worker(rank, world, dims, ranks, iters, seed):
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(ranks)
    us = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
    full = np.einsum("abc,ia,jb,kc->ijk", core, *us) + 1e-3 * rng.standard_normal(dims)
    c0, c1 = slab(dims[2], world, rank)
    t_local = torch.tensor(full[:, :, c0:c1])
    core, u, fits, it = hooi_sharded(t_local, dims, ranks, max_iters=iters, tol=-1.0,
                                     ops=HostOps())
    return {"fits": fits, "iters": it, "u": [x.numpy() for x in u], "core": core.numpy(),
            "full": full}


@pytest.mark.parametrize("dims,world", [((12, 10, 9), 2), ((16, 16, 16), 2), ((9, 10, 13), 2),
                                        ((16, 16, 16), 3)])
def test_hooi_sharded_matches_oracle(dims, world):
    """Sharded HOOI (slab on mode 2, ring-assembled HOSVD Gram, all-reduce /
    all-gather per mode update) equals the single-process oracle; uneven
    slabs at world 3; the non-reuse product order at (9, 10, 13)."""
    from oracle import tucker as otucker
    ranks = (3, 3, 2)
    out = _run(world, _hooi_worker, dims, ranks, 4, 11)
    r0 = out[0][1]
    for _, rk in out[1:]:   # every rank holds the same model
        np.testing.assert_allclose(r0["fits"], rk["fits"], rtol=0, atol=0)
        for a, b in zip(r0["u"], rk["u"]):
            np.testing.assert_array_equal(a, b)
    ref = otucker.hooi(r0["full"], ranks, max_iters=4, tol=-1.0)
    np.testing.assert_allclose(r0["fits"], ref["fit_history"], atol=1e-10)
    for u, ur in zip(r0["u"], ref["factors"]):
        np.testing.assert_allclose(u @ u.T, ur @ ur.T, atol=1e-8)


def _slab_worker(rank, world, cid, ext, seed):
    """Rank r evaluates its slab of one contraction (shard_contraction views
    into the full buffers, the reference planner lowering on the host) and the
    slabs are all-gathered; no collective on the data path itself."""
    from oracle import plan as oplan
    rng = np.random.default_rng(seed)
    case = [c for c in enumerate_cases(2, 3) if c.case_id == cid][0]
    spec = ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
    la, lb, lc = (Layout.packed([ext[l] for l in labs])
                  for labs in (spec.labels_a, spec.labels_b, spec.labels_c))
    A, B = rng.standard_normal(la.size), rng.standard_normal(lb.size)
    C = np.zeros(lc.size)
    sh = shard_contraction(spec, la, lb, lc, world, rank)
    sla, slb, slc = sh.layouts
    local_ext = dict(ext)
    local_ext[sh.label] = sh.stop - sh.start
    oplan.contract(spec.labels_a, spec.labels_b, spec.labels_c, local_ext,
                   A[sh.offsets[0]:], B[sh.offsets[1]:], 1.0, 0.0, C[sh.offsets[2]:],
                   layouts=(sla, slb, slc))
    mine = torch.tensor(C)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    got = sum(p.numpy() for p in parts)     # slabs are disjoint: the sum reassembles C
    want = np.zeros(lc.size)
    oplan.contract(spec.labels_a, spec.labels_b, spec.labels_c, ext, A, B, 1.0, 0.0, want)
    return float(np.abs(got - want).max())


@pytest.mark.parametrize("cid", ["1.1", "1.3", "3.4", "5.2", "6.6"])
def test_shard_contraction_two_processes(cid):
    """world_size 2 (gloo): each rank executes only its slab; the gathered
    slabs equal the full contraction."""
    ext = dict(m=6, n=5, p=9, k=4)
    out = _run(2, _slab_worker, cid, ext, 5)
    assert all(err <= 1e-12 for _, err in out), out


def test_bench_spawns_ranks():
    """bench.py --gpus N outside torchrun starts N ranks itself (the reference
    arm runs on rank 0 only and reports n_gpus = N)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "1", "--warmup", "0", "--n", "16"],
                         capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
