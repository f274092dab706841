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
  tests).  The HOSVD Gram of the sharded mode needs every slab's cross
  products: the slabs travel around a ring (two resident at a time), T is
  never gathered.

Local compute goes through the sm_100a kernels (``DeviceOps``: the tucker
module's mode products, Grams and device-finished factor updates).
``hooi_sharded`` takes an ``ops`` object -- the tests inject ``HostOps``
(torch CPU arithmetic) so the collective logic runs on a CPU-only box with
gloo; the product path never uses it.
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


class DeviceOps:
    """Local work of sharded HOOI on the sm_100a kernels: planned mode
    products, fp64 Grams on the device, the device-finished factor updates
    (``sbt_hooi_factor_*``) and the status kernel -- the single-GPU HOOI's
    own building blocks (``tucker.py``)."""

    def __init__(self):
        from . import tucker as tk
        self.tk = tk

    def mode_product(self, x, u, mode, fast=False):
        return self.tk._mode_product(x, u, mode, True, fast)

    def gram(self, x, r):
        return self.tk.gram_of_unfolding(x, r)

    def as64(self, x):
        import torch
        return x.data if x.dtype == torch.float64 else x.data.to(torch.float64)

    def cross_gram(self, xa, ra, xb, rb, k):
        """Block X_a^T X_b of the last-mode unfolding: xa / xb are (k x ra) /
        (k x rb) column-major fp64 slabs."""
        import torch
        from .kernels import Op, gemm
        out = torch.empty(ra * rb, dtype=torch.float64, device=xa.device)
        gemm(Op.Transpose, Op.Normal, ra, rb, k, 1.0, xa, k, xb, k, 0.0, out, ra)
        return out.reshape(rb, ra).t()

    def factor_init(self, g, rank):
        _, vecs, _ = self.tk.top_eigh(g, rank)
        return self.tk._sign_fix(vecs.contiguous())

    def factor_iter(self, y, r, rank, warm, status, sweeps):
        tk = self.tk
        if tk._ritz_eligible(y.layout.dims[r], rank, warm):
            return tk._factor_device(y, r, rank, warm, status, r, sweeps)
        status[r] = 1
        return tk._factor_from_tensor(y, r, rank, warm=warm)

    def factor_host(self, y, r, rank, warm):
        return self.tk._factor_from_tensor(y, r, rank, warm=warm)

    def new_status(self, order, device):
        import torch
        return torch.zeros(order, dtype=torch.int32, device=device)

    def status(self, core, st):
        import torch
        out = torch.empty(1 + st.numel(), dtype=torch.float64, device=core.device)
        return self.tk._hooi_status(core, st, out).cpu().numpy()

    def sumsq(self, x):
        import torch
        return torch.sum(x.data.to(torch.float64) ** 2).reshape(1)


class HostOps(DeviceOps):
    """The same steps with torch CPU arithmetic, full eigendecompositions and
    no device kernels: lets the gloo tests run the sharded driver's
    collective logic on a CPU-only box.  Never used by the product path."""

    def __init__(self):
        from . import tucker as tk
        self.tk = tk

    def mode_product(self, x, u, mode, fast=False):
        import torch
        from .layout import DenseTensor
        v = x.view()
        out = torch.movedim(torch.tensordot(u.t().to(v.dtype), v, dims=([1], [mode])), 0, mode)
        return DenseTensor.from_array(out, device=x.device)

    def gram(self, x, r):
        import torch
        v = torch.movedim(x.view(), r, 0).reshape(x.layout.dims[r], -1).to(torch.float64)
        return v @ v.t()

    def cross_gram(self, xa, ra, xb, rb, k):
        return xa[:k * ra].reshape(ra, k) @ xb[:k * rb].reshape(rb, k).t()

    def factor_init(self, g, rank):
        _, vecs = self.tk.jacobi_eigh(g)
        return self.tk._sign_fix(vecs[:, :rank].contiguous())

    def factor_iter(self, y, r, rank, warm, status, sweeps):
        status[r] = 1
        return self.factor_host(y, r, rank, warm)

    def factor_host(self, y, r, rank, warm):
        return self.factor_init(self.gram(y, r), rank)

    def status(self, core, st):
        import torch
        nrm = torch.sqrt(torch.sum(core.data.to(torch.float64) ** 2))
        return np.concatenate([[float(nrm)], st.to(torch.float64).numpy()])


def hooi_sharded(t_local, full_dims, ranks, max_iters: int = 50, tol: float = 1e-10,
                 group=None, ops=None):
    """HOOI with T slab-sharded along its last mode (order 3), reference
    tucker.py:136-174 with the same products in the same order.

    ``t_local`` is this rank's slab T[:, :, c0:c1] (``slab(d2, world,
    rank)``) as a packed ``DenseTensor`` (or a logical torch tensor, packed
    here).  Per mode update: products that contract the sharded mode give
    partial sums -> all-reduce (r0 d1 r2 / d0 r1 r2 elements); the one that
    keeps it gives a mode-2-distributed result -> all-gather (r0 r1 d2);
    ||T||^2 -> all-reduce.  T itself is never gathered: the HOSVD Gram of the
    sharded mode is assembled from slab cross products passed around a ring
    (W - 1 point-to-point steps, two slabs resident), then all-gathered as
    d2 x d2 row blocks.  Factor updates run on the replicated partial cores
    with the device-finished sweeps (one flag read per iteration; an
    unconverged factor redoes the iteration on the host-driven path), so every
    rank holds the same model.  Returns (core as a logical tensor, factors,
    fit_history, iterations)."""
    import torch
    import torch.distributed as dist

    from .layout import DenseTensor

    ops = ops or DeviceOps()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    d0, d1, d2 = (int(d) for d in full_dims)
    c0, c1 = slab(d2, world, rank)
    if isinstance(t_local, torch.Tensor):
        t_local = DenseTensor.from_array(t_local, device=t_local.device)
    if tuple(t_local.layout.dims) != (d0, d1, c1 - c0) or not t_local.layout.is_packed():
        raise ValueError(f"rank {rank}: slab {t_local.layout} != packed {(d0, d1, c1 - c0)}")
    ranks = tuple(int(r) for r in ranks)
    if len(ranks) != 3 or not all(1 <= r <= d for r, d in zip(ranks, (d0, d1, d2))):
        raise ValueError(f"invalid ranks {ranks} for dims {full_dims}")
    dev = t_local.device
    sizes = [slab(d2, world, r)[1] - slab(d2, world, r)[0] for r in range(world)]
    starts = [slab(d2, world, r)[0] for r in range(world)]
    mx = max(sizes)

    # gloo (CPU tests, or ranks sharing one GPU) moves CUDA tensors through
    # host copies; NCCL takes them directly
    host_coll = dist.get_backend(group) == "gloo" and dev.type == "cuda"

    def allreduce(x):
        allreduce_t(x.data, group)
        return x

    def allgather_last(x):
        """Packed (a, b, d2) from the ranks' (a, b, slab) pieces: the last
        mode is the slowest, so a slab is one contiguous chunk."""
        a, b, _ = x.layout.dims
        per = a * b
        pad = torch.zeros(per * mx, dtype=x.dtype, device="cpu" if host_coll else x.device)
        pad[:x.data.numel()] = x.data
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        flat = torch.cat([q[:per * s] for q, s in zip(parts, sizes)]).to(x.device)
        return DenseTensor(Layout.packed((a, b, d2)), flat)

    def ring_gram_last(x):
        """d2 x d2 Gram of the mode-2 unfolding without gathering T."""
        k = d0 * d1
        mine = ops.as64(x)
        buf = torch.zeros(k * mx, dtype=torch.float64, device=dev)
        buf[:mine.numel()] = mine
        rows = torch.zeros(mx, d2, dtype=torch.float64, device=dev)
        cl = c1 - c0
        for step in range(world):
            holder = (rank - step) % world
            blk = ops.cross_gram(mine, cl, buf, sizes[holder], k)
            rows[:cl, starts[holder]:starts[holder] + sizes[holder]] = blk
            if step < world - 1:
                sbuf = buf.cpu() if host_coll else buf
                nbuf = torch.empty_like(sbuf)
                reqs = dist.batch_isend_irecv([
                    dist.P2POp(dist.isend, sbuf, (rank + 1) % world, group),
                    dist.P2POp(dist.irecv, nbuf, (rank - 1) % world, group)])
                for q in reqs:
                    q.wait()
                buf = nbuf.to(dev)
        rows_c = rows.cpu() if host_coll else rows
        parts = [torch.empty_like(rows_c) for _ in range(world)]
        dist.all_gather(parts, rows_c, group=group)
        g = torch.cat([q[:s] for q, s in zip(parts, sizes)]).to(dev)
        return 0.5 * (g + g.t())

    def local_u2(u2):
        return u2[c0:c1]

    def chain(factors, skip, fast=False):
        """Reference product order (tucker.py:95-99: larger reduction extent
        first, ties ascending) on the slab; the collective at the end.  fast:
        the result only feeds a factor update (tucker._mode_product)."""
        modes = sorted((m for m in range(3) if m != skip), key=lambda m: -full_dims[m])
        cur, partial = t_local, False
        for m in modes:
            cur = ops.mode_product(cur, local_u2(factors[m]) if m == 2 else factors[m], m, fast)
            partial = partial or m == 2
        return allreduce(cur) if partial else allgather_last(cur)

    # HOSVD initialisation (tucker.py:153-155)
    u = [None, None, None]
    for r in (0, 1):
        u[r] = ops.factor_init(allreduce_t(ops.gram(t_local, r).contiguous(), group), ranks[r])
    u[2] = ops.factor_init(ring_gram_last(t_local), ranks[2])
    norm_t = float(torch.sqrt(allreduce_t(ops.sumsq(t_local), group)))
    reuse = d0 >= d1 and d0 >= d2

    def sweep(factors, factor_fn):
        """One iteration (tucker.py:160-167); returns the core (replicated)."""
        if reuse:
            y = chain(factors, 0, fast=True)
            factors[0] = factor_fn(y, 0, factors[0])
            x0 = ops.mode_product(t_local, factors[0], 0)
            y = allreduce(ops.mode_product(x0, local_u2(factors[2]), 2, fast=True))
            factors[1] = factor_fn(y, 1, factors[1])
            y2 = allgather_last(ops.mode_product(x0, factors[1], 1))
            factors[2] = factor_fn(y2, 2, factors[2])
            if d1 >= d2:
                return ops.mode_product(y2, factors[2], 2)
            g = allreduce(ops.mode_product(x0, local_u2(factors[2]), 2))
            return ops.mode_product(g, factors[1], 1)
        for r in range(3):
            factors[r] = factor_fn(chain(factors, r, fast=True), r, factors[r])
        return chain(factors, None)

    fits, prev, iters = [], -np.inf, 0
    dt = t_local.dtype
    for it in range(max_iters):
        iters = it + 1
        sweeps = 2 if (it == 0 or dt == torch.float64) else 1
        st = ops.new_status(3, dev)
        start = list(u)
        core = sweep(u, lambda y, r, warm: ops.factor_iter(y, r, ranks[r], warm, st, sweeps))
        vals = ops.status(core, st)
        if not np.all(vals[1:] == 1.0):   # identical on every rank (same inputs, same kernels)
            u = start
            core = sweep(u, lambda y, r, warm: ops.factor_host(y, r, ranks[r], warm))
            vals = ops.status(core, st)
        resid = np.sqrt(max(0.0, norm_t ** 2 - float(vals[0]) ** 2))
        fit = 1.0 - resid / norm_t if norm_t > 0 else 1.0
        fits.append(fit)
        if fit - prev < tol and it > 0:
            break
        prev = fit
    return core.view(), u, fits, iters


def allreduce_t(x, group=None):
    """In-place sum over the group (through a host copy for CUDA tensors on
    gloo)."""
    import torch.distributed as dist
    if x.is_cuda and dist.get_backend(group) == "gloo":
        h = x.cpu()
        dist.all_reduce(h, group=group)
        x.copy_(h)
    else:
        dist.all_reduce(x, group=group)
    return x
