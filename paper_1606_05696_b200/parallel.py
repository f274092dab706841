"""Multi-GPU execution: one process per GPU, ``torch.distributed`` for plumbing.

Two regimes, following SURVEY.md section 8e:

* **Batch / free-mode sharding (no collective).**  A single-index contraction
  whose output has a free mode owned by one operand partitions along that
  mode: rank r holds a contiguous slab of that operand and of C, the other
  operand is replicated, and each rank runs the SAME planned contraction on
  its slab (one launch, zero communication).  ``shard_contraction`` returns the
  rank's slab layouts and element offsets; ``slab`` the index range.

* **Tucker / HOOI (one exchange per mode update).**  T is slab-sharded along
  its last mode (contiguous in column-major storage).  Products that contract
  the sharded mode produce partial sums -> all-reduce; products that keep it
  produce a mode-distributed result -> all-gather; norms -> all-reduce.  The
  collectives are NCCL over NVLink on GPU tensors (gloo on CPU tensors in the
  tests).  The HOSVD initialisation of the sharded mode needs every slab's
  cross products, so it all-gathers T once.

Local compute goes through the sm_100a kernels (``paper_1606_05696_b200.tucker``
mode products).  ``hooi_sharded`` takes an optional ``local`` hook -- the
tests inject a CPU einsum implementation so the collective logic runs on a
CPU-only box with gloo; the product path never uses it.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .layout import Layout
from .notation import ContractionSpec


def slab(n: int, world: int, rank: int):
    """Contiguous [start, stop) block of ``n`` indices for ``rank`` (balanced:
    the first n % world ranks get one extra index)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    q, r = divmod(n, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


@dataclass(frozen=True)
class ShardedOperands:
    label: str                  # sharded free label
    start: int
    stop: int
    layouts: tuple              # (la, lb, lc) of the rank's slab views
    offsets: tuple              # element offsets of the slab views into the full buffers


def shard_contraction(spec: ContractionSpec, la: Layout, lb: Layout, lc: Layout,
                      world: int, rank: int, label: str | None = None) -> ShardedOperands:
    """Slab of a single-index contraction along a free label (default: C's
    last mode).  The label must appear in C and in exactly one operand, so the
    slabs are independent (no reduction, no collective)."""
    if not spec.labels_c:
        raise ValueError("scalar contractions do not shard")
    label = label or spec.labels_c[-1]
    if label not in spec.labels_c:
        raise ValueError(f"label {label!r} is not a free (output) label")
    in_a, in_b = label in spec.labels_a, label in spec.labels_b
    if in_a == in_b:
        raise ValueError(f"label {label!r} must belong to exactly one operand")
    ext = dict(zip(spec.labels_c, lc.dims))[label]
    start, stop = slab(ext, world, rank)

    def cut(labels, lay):
        if label not in labels:
            return lay, 0
        i = labels.index(label)
        dims = list(lay.dims)
        dims[i] = stop - start
        return Layout(tuple(dims), lay.strides), start * lay.strides[i]

    (la2, oa), (lb2, ob), (lc2, oc) = (cut(spec.labels_a, la), cut(spec.labels_b, lb),
                                       cut(spec.labels_c, lc))
    return ShardedOperands(label, start, stop, (la2, lb2, lc2), (oa, ob, oc))


# ----------------------------------------------------------------------------- Tucker


def _device_local():
    """Local kernels: logical torch tensors in, device sm_100a contractions."""
    from . import tucker as tk
    from .layout import DenseTensor

    def to_dense(x):
        import torch
        flat = x.permute(*reversed(range(x.dim()))).contiguous().reshape(-1)
        return DenseTensor(Layout.packed(tuple(x.shape)), flat)

    def from_dense(t):
        return t.view()

    def mode_product(x, u, mode):
        return from_dense(tk._mode_product(to_dense(x), u, mode, True))

    def gram(x, mode):
        return tk.gram_of_unfolding(to_dense(x), mode)

    return mode_product, gram


def _einsum_local():
    """Reference-free CPU implementation used by the gloo tests only."""
    import torch

    def mode_product(x, u, mode):
        out = torch.tensordot(u.t().to(x.dtype), x, dims=([1], [mode]))
        return torch.movedim(out, 0, mode)

    def gram(x, mode):
        m = torch.movedim(x, mode, 0).reshape(x.shape[mode], -1).to(torch.float64)
        return m @ m.t()

    return mode_product, gram


def _factor(gram, rank, warm=None, dtype="float64"):
    """Top-``rank`` sign-fixed eigenvectors of an (all-reduced, hence
    rank-identical) Gram: the device subspace solver for CUDA Grams, the full
    eigendecomposition for the CPU (gloo test) path."""
    from .tucker import _SUBSPACE_TOL, _SUBSPACE_TOL_F32, _sign_fix, jacobi_eigh, top_eigh
    if gram.is_cuda:
        tol = _SUBSPACE_TOL if dtype == "float64" else _SUBSPACE_TOL_F32
        _, vecs, _ = top_eigh(gram, rank, q0=warm, tol=tol)
    else:
        _, vecs = jacobi_eigh(gram)
        vecs = vecs[:, :rank]
    return _sign_fix(vecs.contiguous())


def hooi_sharded(t_local, full_dims, ranks, max_iters: int = 50, tol: float = 1e-10,
                 group=None, local=None):
    """HOOI with T slab-sharded along its last mode (order 3).

    ``t_local`` is this rank's slab T[:, :, c0:c1] as a logical torch tensor
    (CUDA for the product path).  Returns (core, factors, fit_history,
    iterations), identical on every rank.  Same algorithm and product order as
    ``tucker.hooi`` (reference tucker.py:136-174)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    d0, d1, d2 = full_dims
    c0, c1 = slab(d2, world, rank)
    if tuple(t_local.shape) != (d0, d1, c1 - c0):
        raise ValueError(f"rank {rank}: slab shape {tuple(t_local.shape)} != "
                         f"{(d0, d1, c1 - c0)}")
    mode_product, gram = local() if local else _device_local()
    dt = str(t_local.dtype).replace("torch.", "")
    ranks = tuple(int(r) for r in ranks)

    def allreduce(x):
        dist.all_reduce(x, group=group)
        return x

    def allgather_last(x):
        """Concatenate the ranks' slabs along the last mode (uneven slabs ok)."""
        sizes = [slab(d2, world, r)[1] - slab(d2, world, r)[0] for r in range(world)]
        mx = max(sizes)
        pad = torch.zeros(x.shape[:-1] + (mx,), dtype=x.dtype, device=x.device)
        pad[..., :x.shape[-1]] = x
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad.contiguous(), group=group)
        return torch.cat([p[..., :s] for p, s in zip(parts, sizes)], dim=-1)

    # HOSVD init: modes 0/1 Grams are sums over slabs; the sharded mode needs
    # the cross-slab products, so gather T once.
    u = [None, None, None]
    for r in (0, 1):
        u[r] = _factor(allreduce(gram(t_local, r).contiguous()), ranks[r])
    t_full = allgather_last(t_local)
    u[2] = _factor(gram(t_full, 2), ranks[2])
    del t_full
    nt2 = allreduce(torch.sum(t_local.to(torch.float64) ** 2).reshape(1))
    norm_t = float(torch.sqrt(nt2))
    u2_local = lambda: u[2][c0:c1]  # noqa: E731

    fits, prev, iters = [], -np.inf, 0
    for it in range(max_iters):
        iters = it + 1
        # skip=0: modes 1 then 2 (contracting the sharded mode: partial sums)
        y = allreduce(mode_product(mode_product(t_local, u[1], 1), u2_local(), 2).contiguous())
        u[0] = _factor(gram(y, 0), ranks[0], u[0], dt)
        x0 = mode_product(t_local, u[0], 0)
        # skip=1: [0, 2] -> partial sums over the sharded mode
        y = allreduce(mode_product(x0, u2_local(), 2).contiguous())
        u[1] = _factor(gram(y, 1), ranks[1], u[1], dt)
        # skip=2: [0, 1] -> mode-2 distributed result
        y2 = allgather_last(mode_product(x0, u[1], 1).contiguous())
        u[2] = _factor(gram(y2, 2), ranks[2], u[2], dt)
        core = mode_product(y2, u[2], 2)
        g2 = float(torch.sum(core.to(torch.float64) ** 2))
        resid = np.sqrt(max(0.0, norm_t ** 2 - g2))
        fit = 1.0 - resid / norm_t if norm_t > 0 else 1.0
        fits.append(fit)
        if fit - prev < tol and it > 0:
            break
        prev = fit
    return core, u, fits, iters
