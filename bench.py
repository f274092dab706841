#!/usr/bin/env python
"""Benchmark: single-index tensor-contraction throughput on B200 (BASELINE.json).

Default line (the driver's headline): the sweep of all 36 second-order x
third-order single-index contraction cases at n = 256 in fp64 -- the
reference's own precision (``layout.py:149-150``) -- each planned with the
reference's dispatcher semantics and executed on the sm_100a kernels.

    python bench.py [--gpus N] [--steps K] [--warmup W]            # sweep, fp64, n=256
    python bench.py --config c1|sweep|small|order4|hooi|conventional [--dtype f32|f64] [--n N]
    python bench.py --impl reference ...   # the reference algorithm on the host CPU

Configs (BASELINE.json ``configs``):
  c1      configs[0]: strided_batched_gemm('N','N',256,256,256,1,A,256,0,B,256,65536,0,C,256,65536,256)
  sweep   configs[1]: all 36 cases at extent n (default 256)
  small   configs[2]: batched GEMM n = 8..64, P = 10^6 per GPU (headline n = 32)
  hooi    configs[3]: Tucker HOOI 512^3, rank 32, fp32
  order4  configs[4]: C[mnpq] = A[mkp] B[nkq], n = 128 (one nested-batched launch)

Multi-GPU: ``--gpus N`` without a torchrun environment re-launches itself as N
ranks (one process per GPU, NCCL).  Every config partitions along a batch /
free mode with no data-path collective, so scaling is
WEAK: rank r holds shard r of a problem N times the single-GPU one (the p-slab
of C's last mode for the sweep / C1, the batch range for small, the q-slab for
order4); HOOI slab-shards one T along mode 2 (all-reduce / all-gather per mode
update, strong scaling).  value = work of all ranks / max-over-ranks device time.

Every line carries ``roofline`` (dominant kernel, event-timed on its launching
stream), ``cpu_baseline`` (the oracle port on the host cores, rank 0 at N = 1:
all-core and serial), ``e2e`` (the same metric through the reference-facing
host-buffer seam, ``backend.batched_core`` over pinned numpy buffers, host <->
device copies inside the timed region), ``gpu_launches`` and ``clocks``.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "contraction GFLOP/s and % roofline vs n (1/2/4/8 B200) next to CPU ref"
EXCEPTIONAL_CASES = {"3.4", "3.6", "4.4", "4.6", "5.4", "5.6", "6.4", "6.6"}
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}
FP64_NOMINAL_TFLOPS = 37.0  # HGX B200 datasheet FP64 / FP64 tensor core
DEFAULT_DTYPE = {"sweep": "f64", "c1": "f64", "small": "f32", "order4": "f64", "hooi": "f32",
                 "conventional": "f64"}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return dict(FALLBACK_PEAKS)


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def case_shapes(n):
    from paper_1606_05696_b200.planner import enumerate_cases
    return [(case, dict(m=n, n=n, p=n, k=n)) for case in enumerate_cases(2, 3)]


def flops_bytes(n, itemsize):
    """Algorithmic FLOPs and bytes of one case at extent n (beta = 0): A is
    n^2, B and C are n^3."""
    return 2.0 * n ** 4, itemsize * (n * n + 2.0 * n ** 3)


# ----------------------------------------------------------------------------- clocks


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML every ~5 ms while the
    timed region runs (the B200_PROFILING clocks line, without nvidia-smi's
    ~100 ms start-up latency)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - no NVML
            self._nv = None
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.03)  # sampler running before the timed region starts
        return self

    def _run(self):
        nv = self._nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM),
                                     int(get_reasons(self._h))))
            except Exception:
                pass
            time.sleep(0.005)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = sorted(name for name, bit in self.REASONS.items()
                         if any(r & bit for _, r in self.samples))
        return {"sm_mhz": statistics.median(c for c, _ in self.samples),
                "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml"}


# ----------------------------------------------------------------------------- ranks


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args) -> int:
    """``--gpus N`` outside torchrun: start N ranks of this script (one process
    per GPU, the torchrun environment variables set), pass rank 0's output
    through, return the worst exit code."""
    import torch
    n = args.gpus
    share = os.environ.get("SBT_SHARE_GPU") == "1"   # test hook: N ranks on one GPU (gloo)
    if args.impl != "reference" and not share and torch.cuda.device_count() < n:
        raise SystemExit(f"--gpus {n}: only {torch.cuda.device_count()} CUDA device(s) visible")
    port = _free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        out = None if r == 0 else subprocess.DEVNULL
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve())] + sys.argv[1:],
                                      env=env, stdout=out))
    return max(p.wait() for p in procs)


class Ctx:
    """This process's rank, world and device (torch.distributed when world > 1)."""

    def __init__(self):
        import torch
        import torch.distributed as dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        share = os.environ.get("SBT_SHARE_GPU") == "1"
        self.device = torch.device("cuda", 0 if share else self.local)
        torch.cuda.set_device(self.device)
        self.backend = None
        if self.world > 1:
            self.backend = os.environ.get("SBT_DIST_BACKEND", "gloo" if share else "nccl")
            kw = {"device_id": self.device} if self.backend == "nccl" else {}
            dist.init_process_group(self.backend, **kw)
        self.dist = dist

    def barrier(self):
        if self.world > 1:
            if self.backend == "nccl":
                self.dist.barrier(device_ids=[self.device.index])
            else:
                self.dist.barrier()

    def max_over_ranks(self, x: float) -> float:
        import torch
        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64,
                         device=self.device if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1 and self.dist.is_initialized():
            self.dist.destroy_process_group()


def capture(fn, device):
    """Capture fn() (launch-only work on the current stream) as a CUDA graph;
    returns (graph, library launches per replay)."""
    import torch
    from paper_1606_05696_b200 import _lib
    stream = torch.cuda.current_stream(device)
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(device)
    cap.wait_stream(stream)
    n0 = _lib.launch_count()
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            fn()
    stream.wait_stream(cap)
    return g, _lib.launch_count() - n0


def timed_steps(ctx, fn, steps, warmup, launches_per_step):
    """W warm-up steps, then EXACTLY K timed steps bracketed by a barrier and a
    device synchronize on both sides, CUDA events on the launching stream, NVML
    clocks sampled during the region; returns (max-over-ranks ms per step,
    clocks, launches in the timed region)."""
    import torch
    from paper_1606_05696_b200 import _lib
    stream = torch.cuda.current_stream(ctx.device)
    for _ in range(warmup):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ctx.barrier()
    torch.cuda.synchronize()
    n0 = _lib.launch_count()
    with ClockSampler(ctx.device.index) as clocks:
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = _lib.launch_count() - n0 or launches_per_step * steps
    ctx.barrier()
    ms = ctx.max_over_ranks(e0.elapsed_time(e1)) / steps
    return ms, clocks.summary(), launches


def event_ms(fn, reps, device):
    """Mean device time of fn() (a launch, or a graph replay) with CUDA events
    on the launching stream, after one untimed call."""
    import torch
    stream = torch.cuda.current_stream(device)
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def ncu_traffic(key):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel from a committed ncu --set full capture (profiles/ncu_traffic.json)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(key)
    except ValueError:
        return None


def tensor_peak(dtype_name, sustained=False):
    """(TFLOP/s, note): fp32 = 3xTF32 = measured tcgen05 kind::tf32 dense peak / 3;
    fp64 = measured DMMA peak (both probed in-run by the library)."""
    from paper_1606_05696_b200 import _lib
    if dtype_name == "f32":
        try:
            if sustained:
                v = _lib.probe_tf32_sustained(3.0)
                return v / 3.0, (f"3xTF32 = sustained tcgen05 TF32 peak {v:.0f} TFLOP/s / 3 "
                                 "(sbt_probe_tf32_sustained, 3 s back to back: power-capped clock)")
            v = _lib.probe_tf32_peak()
            return v / 3.0, (f"3xTF32 = measured tcgen05 TF32 dense peak {v:.0f} TFLOP/s / 3 "
                             "(sbt_probe_tf32_peak, in-run, burst)")
        except Exception:
            bf = load_peaks().get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"])
            return bf / 2.0 / 3.0, "3xTF32 = bf16_tflops / 2 / 3 (probe failed)"
    try:
        return _lib.probe_fp64_peak("dmma"), "fp64 DMMA measured in-run (sbt_probe_fp64_peak)"
    except Exception:
        return FP64_NOMINAL_TFLOPS, "fp64 DMMA nominal (datasheet 37 TFLOP/s)"


def roofline_obj(flops, nbytes, ms, tpeak, tnote, hbm, kernel, traffic_key, extra=None,
                 traffic_scale=1):
    """roofline of one kernel: bound = the slower of tensor pipe at peak and
    algorithmic bytes at HBM bandwidth; achieved in the bound's unit.
    traffic_scale: the ncu capture covers one of that many identical launches
    that the timed "launch" stands for (fp64 sweep: one DMMA launch per case)."""
    t_tensor = flops / (tpeak * 1e12)
    t_hbm = nbytes / (hbm * 1e9)
    bound = "tensor" if t_tensor >= t_hbm else "hbm"
    if bound == "tensor":
        achieved, peak, unit = flops / (ms * 1e-3) / 1e12, tpeak, "TFLOP/s"
    else:
        achieved, peak, unit = nbytes / (ms * 1e-3) / 1e9, hbm, "GB/s"
    out = {"bound": bound, "kernel": kernel, "achieved": round(achieved, 3),
           "peak": round(peak, 2), "unit": unit, "frac": round(achieved / peak, 4),
           "traffic": (ncu_traffic(traffic_key) * traffic_scale
                       if ncu_traffic(traffic_key) is not None else None),
           "peak_source": tnote if bound == "tensor" else
           load_peaks()["source"], "launch_ms": round(ms, 4),
           "algorithmic": {"flop": flops, "bytes": nbytes},
           "hbm_achieved_gbs": round(nbytes / (ms * 1e-3) / 1e9, 1), "hbm_peak_gbs": hbm,
           "tensor_peak_tflops": round(tpeak, 2)}
    if extra:
        out.update(extra)
    return out


def pinned_np(numel, dtype, fill=True, seed=0):
    """A numpy view of a page-locked torch host buffer (the host seam DMAs it
    directly), filled with U[-1,1]."""
    import torch
    t = torch.empty(numel, dtype=dtype, pin_memory=True)
    if fill:
        g = torch.Generator().manual_seed(seed)
        t.uniform_(-1, 1, generator=g)
    return t, t.numpy()


# ----------------------------------------------------------------------------- CPU baseline


def _timed_cpu(fn, threads):
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        fn()
        return time.perf_counter() - t0


def cpu_baseline_obj(flops, fn, sample, scale=1.0, serial=True):
    """The oracle port (the reference numpy backend's algorithm: planner
    lowering + numpy/OpenBLAS cores, fp64) on the host: all host threads, and
    one thread (the paper's serial protocol).  ``flops`` = work of one fn()
    call; ``scale`` converts the sample's rate to the metric unit."""
    cores = os.cpu_count() or 1
    fn()  # warm-up (BLAS threads, page faults)
    dt = _timed_cpu(fn, cores)
    out = {"value": round(flops / dt / 1e9 * scale, 3), "unit": "GFLOP/s", "cores": cores,
           "kind": "port", "sample": f"{sample} ({dt:.2f} s)", "cpu_model": cpu_model(),
           "impl": "oracle/ (numpy restatement of the reference cores + dispatcher lowering; "
                   "numpy/OpenBLAS, fp64)"}
    if serial:
        ds = _timed_cpu(fn, 1)
        out["serial"] = {"value": round(flops / ds / 1e9 * scale, 3), "cores": 1,
                         "seconds": round(ds, 2)}
    return out


def cpu_sweep(n, dtype_name, cases=None):
    """One oracle-port pass over the 36-case sweep at extent n (fp64 arithmetic
    on the fp32- or fp64-valued inputs)."""
    from oracle import plan as oplan
    from paper_1606_05696_b200.planner import enumerate_cases  # case catalogue only
    rng = np.random.default_rng(0)
    src = np.float32 if dtype_name == "f32" else np.float64
    a = rng.uniform(-1, 1, n * n).astype(src).astype(np.float64)
    b = rng.uniform(-1, 1, n ** 3).astype(src).astype(np.float64)
    c = np.empty(n ** 3)
    todo = [c for c in enumerate_cases(2, 3) if cases is None or c.case_id in cases]

    def run():
        for case in todo:
            x = a if len(case.labels_a) == 2 else b
            y = a if len(case.labels_b) == 2 else b
            oplan.contract(case.labels_a, case.labels_b, case.labels_c,
                           dict(m=n, n=n, p=n, k=n), x, y, 1.0, 0.0, c)
    return run, len(todo) * 2.0 * n ** 4, len(todo)


# ----------------------------------------------------------------------------- sweep (configs[1])


def build_sets(cases, n, dtype, device, nsets, seed, distinct_c=False):
    import torch
    from paper_1606_05696_b200.layout import DenseTensor, Layout
    from paper_1606_05696_b200.notation import ContractionSpec
    from paper_1606_05696_b200.planner import plan_single_mode
    g = torch.Generator(device=device).manual_seed(seed)
    size_a, size_b = n * n, n ** 3
    sets = []
    for s in range(nsets):
        a = (torch.rand(size_a, generator=g, device=device, dtype=dtype) * 2 - 1)
        b = (torch.rand(size_b, generator=g, device=device, dtype=dtype) * 2 - 1)
        c = torch.empty(size_b, device=device, dtype=dtype)
        sets.append((a, b, c))
    work = []
    for i, (case, ext) in enumerate(cases):
        la = Layout.packed([ext[l] for l in case.labels_a])
        lb = Layout.packed([ext[l] for l in case.labels_b])
        lc = Layout.packed([ext[l] for l in case.labels_c])
        plan = plan_single_mode(ContractionSpec(case.labels_a, case.labels_b, case.labels_c),
                                la, lb, lc)
        a, b, c = sets[i % nsets]
        if distinct_c:  # grouped execution: every case writes its own C
            c = torch.empty(size_b, device=device, dtype=dtype)
        # the order-2 operand may be A or B of the case: bind buffers by size
        ta = DenseTensor(la, a if la.size == size_a else b)
        tb = DenseTensor(lb, a if lb.size == size_a else b)
        work.append((case.case_id, plan, ta, tb, DenseTensor(lc, c)))
    return work


def shard_note(n, world, rank, label_desc):
    from paper_1606_05696_b200.parallel import slab
    s0, s1 = slab(n * world, world, rank)
    return (f"weak: rank r holds slab [r*{n}, (r+1)*{n}) of {label_desc} (global extent "
            f"{n * world}, parallel.slab / shard_contraction), stored packed; the operand "
            f"without that mode is replicated; no collective (rank {rank}: [{s0}, {s1}))")


def seam_call(plan, a_np, b_np, c_np, alpha=1.0, beta=0.0):
    """One planned contraction through the reference-facing host-buffer seam:
    the plan's lowered strided-core call (reference planner.py:508-581 ->
    kernels.py -> backend.batched_core) on numpy buffers -- H2D of the touched
    operand spans, one sm_100a launch, D2H of C, synchronise."""
    from paper_1606_05696_b200 import backend
    from paper_1606_05696_b200.planner import lower_plan
    L = lower_plan(plan)
    x, y = (a_np, b_np) if L.first == "A" else (b_np, a_np)
    ars, acs, apt, apt2, brs, bcs, bpt, bpt2, crs, ccs, cpt, cpt2 = L.strides
    for ox, oy, oc in L.outer:
        for q in range(L.batch2):
            backend.batched_core(L.m, L.n, L.k, alpha, x, ox + q * apt2, ars, acs, apt,
                                 y, oy + q * bpt2, brs, bcs, bpt, beta, c_np, oc + q * cpt2,
                                 crs, ccs, cpt, L.batch)


def run_sweep(args, ctx):
    import torch
    from paper_1606_05696_b200 import _lib
    from paper_1606_05696_b200.planner import execute_plan, execute_plans
    dev = ctx.device
    dtype = torch.float32 if args.dtype == "f32" else torch.float64
    itemsize = 4 if args.dtype == "f32" else 8
    n = args.n
    tpeak, tnote = tensor_peak(args.dtype)       # before heavy work: burst clocks
    if args.dtype == "f32" and n >= 512:
        tpeak, tnote = tensor_peak(args.dtype, sustained=True)
    cases = case_shapes(n)
    # grouped: the step's 36 independent contractions as ONE execute_plans call
    # (one persistent launch per kernel configuration); every case then needs
    # its own C.  n >= 512: cases are >= 0.5 ms, per-launch overheads vanish.
    group = (not args.no_group) and n <= 256
    nsets = 4
    work = build_sets(cases, n, dtype, dev, nsets, seed=1234 + ctx.rank, distinct_c=group)
    kernel_of = {}
    for cid, plan, a, b, c in work:           # one untimed pass: kernel families
        execute_plan(plan, a, b, 1.0, 0.0, c)
        kernel_of[cid] = _lib.last_kernel()
    # per-case attribution (events between launches, no graph)
    per_case = {}
    for cid, plan, a, b, c in work:   # device time of one call (graph replay: no host gaps)
        g1, _ = capture(lambda: execute_plan(plan, a, b, 1.0, 0.0, c), dev)
        per_case[cid] = event_ms(g1.replay, 5, dev)
        del g1
    fl, by = flops_bytes(n, itemsize)
    # dominant kernel: one grouped launch per subset, event-timed on its stream
    fam = {}
    if group:
        for name, sub in (("plain", [w for w in work if w[0] not in EXCEPTIONAL_CASES]),
                          ("exceptional", [w for w in work if w[0] in EXCEPTIONAL_CASES])):
            calls = [(plan, a, b, 1.0, 0.0, c) for cid, plan, a, b, c in sub]
            g, _ = capture(lambda: execute_plans(calls), dev)
            ms = event_ms(g.replay, max(3, args.steps), dev)
            fam[name] = {"cases": len(sub), "ms": ms, "kernel": _lib.last_kernel()}
    else:
        for cid, ms in per_case.items():
            k = kernel_of[cid]
            f = fam.setdefault(k, {"cases": 0, "ms": 0.0, "kernel": k})
            f["cases"] += 1
            f["ms"] += ms

    def issue_step():
        if group:
            execute_plans([(plan, a, b, 1.0, 0.0, c) for cid, plan, a, b, c in work])
        else:
            for cid, plan, a, b, c in work:
                execute_plan(plan, a, b, 1.0, 0.0, c)

    graph, lps = capture(issue_step, dev)
    ms, clocks, launches = timed_steps(ctx, graph.replay, args.steps, args.warmup, lps)
    step_flops = fl * len(work)
    value = step_flops * ctx.world / (ms * 1e-3) / 1e9
    hbm = load_peaks().get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"])
    dom = max(fam, key=lambda k: fam[k]["ms"])
    d = fam[dom]
    # fp32 groups are ONE persistent launch over all their cases; fp64 groups
    # are one DMMA launch per case (forked over streams): the committed ncu
    # capture is then of one case's launch
    per_case_launch = not d["kernel"].startswith("tc_tf32x3_pair")
    roof = roofline_obj(d["cases"] * fl, d["cases"] * by, d["ms"], tpeak, tnote, hbm,
                        d["kernel"], f"{d['kernel']}/n{n}/{args.dtype}",
                        traffic_scale=d["cases"] if per_case_launch else 1, extra={
                            "traffic_note": ("ncu dram bytes of one case's launch x the cases"
                                             if per_case_launch else
                                             "ncu dram bytes of the grouped launch"),
                            "per_launch_cases": d["cases"],
                            "kernel_share_of_step": round(d["ms"] / sum(
                                f["ms"] for f in fam.values()), 4),
                            "step_frac_of_roofline": round(
                                max(step_flops / (tpeak * 1e12), len(work) * by / (hbm * 1e9))
                                * 1e3 / ms, 4),
                            "algorithmic_note": "per case: 2n^4 FLOP; s*(n^2 + 2n^3) B (A, B "
                                                "read once, C written once, beta = 0) x the "
                                                "cases one launch processes",
                            "measured_in": "CUDA events on the launching stream around the "
                                           "dominant grouped launch (CUDA graph replay)"})
    line = base_line(args, ctx, value, ms, launches, clocks)
    line["config"] = {"workload": f"36-case single-index sweep (configs[1]) at n={n}",
                      "n": n, "cases": len(work),
                      "gflop_per_step_per_gpu": round(step_flops / 1e9, 2),
                      "parallelism": f"dp{ctx.world} (batch/free-mode shards)",
                      "sharding": shard_note(n, ctx.world, ctx.rank, "C's last mode (and the "
                                             "operand that owns it)"),
                      "l2": f"{nsets} rotating operand sets, each > L2 (126 MB)" if n >= 256 else
                            f"{nsets} rotating operand sets; at n={n} the working set fits L2 "
                            "(inputs L2-warm)",
                      "issue": ("one execute_plans call per step (grouped persistent launches: "
                                "plain / exceptional), CUDA graph" if group else
                                "36 launches per step, CUDA graph"),
                      "alpha": 1.0, "beta": 0.0}
    line["roofline"] = roof
    line["group_launches"] = {k: {"cases": v["cases"], "ms": round(v["ms"], 4),
                                  "kernel": v["kernel"],
                                  "tflops": round(v["cases"] * fl / (v["ms"] * 1e-3) / 1e12, 2)}
                              for k, v in fam.items()}
    line["per_case"] = {cid: {"ms": round(per_case[cid], 4), "kernel": kernel_of[cid],
                              "tflops": round(fl / (per_case[cid] * 1e-3) / 1e12, 2)}
                        for cid in per_case}
    if not args.no_e2e:
        line["e2e"] = e2e_sweep(args, ctx, work, n, dtype, itemsize, step_flops)
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        run, cfl, nc = cpu_sweep(n, args.dtype)
        line["cpu_baseline"] = cpu_baseline_obj(
            cfl, run, f"all {nc} cases at n={n}, fp64 arithmetic on "
                      f"{'fp32-rounded ' if args.dtype == 'f32' else ''}inputs")
    emit(ctx, line)


def e2e_sweep(args, ctx, work, n, dtype, itemsize, step_flops):
    """The sweep through the reference-facing host seam: every case is the
    plan's strided-core call on numpy buffers (backend.batched_core, what the
    reference's kernels.py calls) -- H2D of its operand spans, one launch, D2H
    of C.  Operands live in pinned host memory; the 36 calls are spread over 4
    host threads (the reference's ``threads`` batch chunks; the seam keeps a
    stream and staging per thread, so copies in both directions overlap)."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    size_a, size_b = n * n, n ** 3
    _, ha = pinned_np(size_a, dtype, seed=11 + ctx.rank)
    _, hb = pinned_np(size_b, dtype, seed=12 + ctx.rank)
    nthr = 4
    hcs = [pinned_np(size_b, dtype, fill=False)[1] for _ in range(nthr)]
    jobs = []
    for cid, plan, a, b, c in work:
        ta = ha if a.layout.size == size_a else hb
        tb = ha if b.layout.size == size_a else hb
        jobs.append((plan, ta, tb))

    def worker(t):
        torch.cuda.set_device(ctx.device)
        for plan, ta, tb in jobs[t::nthr]:
            seam_call(plan, ta, tb, hcs[t])

    pool = ThreadPoolExecutor(nthr)

    def step():
        list(pool.map(worker, range(nthr)))

    step()  # warm-up: per-thread streams, arenas, staging
    steps = max(1, min(args.steps, 3))
    ctx.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = ctx.max_over_ranks(time.perf_counter() - t0) / steps
    pool.shutdown()
    h2d = sum(itemsize * (p.layout_a.size + p.layout_b.size) for p, _, _ in jobs)
    d2h = itemsize * size_b * len(jobs)
    return {"value": round(step_flops * ctx.world / dt / 1e9, 2), "unit": "GFLOP/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": round(dt * 1e3, 2), "steps": steps,
            "api": "backend.batched_core (the reference's arithmetic seam) on pinned numpy "
                   "buffers: per case H2D of A and B, one launch, D2H of C, sync; 4 host "
                   "threads (kernels.py threads chunks)"}


# ----------------------------------------------------------------------------- c1 (configs[0])


def run_c1(args, ctx):
    """configs[0]: C[m,n,p] = A[m,k] B[k,n,p] as ONE StridedBatchedGemm call,
    m = n = k = p = 256 (``kernels.py:156-176``)."""
    import torch
    from paper_1606_05696_b200 import _lib
    from paper_1606_05696_b200 import kernels as K
    dev = ctx.device
    dtype = torch.float32 if args.dtype == "f32" else torch.float64
    it = 4 if args.dtype == "f32" else 8
    n = 256
    tpeak, tnote = tensor_peak(args.dtype)
    g = torch.Generator(device=dev).manual_seed(100 + ctx.rank)
    sets = []
    for _ in range(2):    # 2 rotating sets: B + C = 268 MB (fp64) per set > L2
        a = torch.rand(n * n, generator=g, device=dev, dtype=dtype) * 2 - 1
        b = torch.rand(n ** 3, generator=g, device=dev, dtype=dtype) * 2 - 1
        sets.append((a, b, torch.empty(n ** 3, device=dev, dtype=dtype)))

    def call(s):
        a, b, c = s
        K.strided_batched_gemm("N", "N", n, n, n, 1.0, a, n, 0, b, n, n * n, 0.0, c, n, n * n, n)

    call(sets[0])
    kernel = _lib.last_kernel()
    ms_launch = event_ms(lambda: call(sets[0]), max(5, args.steps), dev)
    graph, lps = capture(lambda: [call(s) for s in sets], dev)
    ms2, clocks, launches = timed_steps(ctx, graph.replay, args.steps, args.warmup, lps)
    ms = ms2 / 2       # a graph replay is 2 calls (one per operand set)
    fl = 2.0 * n ** 4
    nbytes = it * (n * n + 2 * n ** 3)
    hbm = load_peaks().get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"])
    line = base_line(args, ctx, fl * ctx.world / (ms * 1e-3) / 1e9, ms, launches // 2, clocks)
    line["steps_note"] = "a step is one C1 call; each timed graph replay runs 2 (2 operand sets)"
    line["config"] = {"workload": "configs[0]: strided_batched_gemm('N','N',256,256,256,1,A,256,"
                                  "0,B,256,65536,0,C,256,65536,256) (C[mnp] = A[mk] B[knp])",
                      "n": n, "parallelism": f"dp{ctx.world}",
                      "sharding": shard_note(n, ctx.world, ctx.rank, "the batch mode p"),
                      "l2": "2 rotating operand sets, B + C > L2 each"}
    line["roofline"] = roofline_obj(fl, nbytes, ms_launch, tpeak, tnote, hbm, kernel,
                                    f"{kernel}/c1/{args.dtype}")
    if not args.no_e2e:
        _, ha = pinned_np(n * n, dtype, seed=1)
        _, hb = pinned_np(n ** 3, dtype, seed=2)
        _, hc = pinned_np(n ** 3, dtype, fill=False)

        def host_call():   # kernels.py:174 -> _run_batched -> backend.batched_core
            K.strided_batched_gemm("N", "N", n, n, n, 1.0, ha, n, 0, hb, n, n * n, 0.0, hc, n,
                                   n * n, n)
        host_call()
        reps = max(3, min(args.steps, 10))
        ctx.barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            host_call()
        dt = ctx.max_over_ranks(time.perf_counter() - t0) / reps
        line["e2e"] = {"value": round(fl * ctx.world / dt / 1e9, 2), "unit": "GFLOP/s",
                       "h2d_bytes_per_step": it * (n * n + n ** 3),
                       "d2h_bytes_per_step": it * n ** 3, "ms_per_step": round(dt * 1e3, 3),
                       "api": "kernels.strided_batched_gemm on pinned numpy buffers (host seam "
                              "sbt_batched_core_host: H2D A, B; launch; D2H C; sync)"}
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        from oracle import cores
        rng = np.random.default_rng(0)
        src = np.float32 if args.dtype == "f32" else np.float64
        A = rng.uniform(-1, 1, n * n).astype(src).astype(np.float64)
        B = rng.uniform(-1, 1, n ** 3).astype(src).astype(np.float64)
        C = np.empty(n ** 3)
        fn = lambda: cores.batched_core(n, n, n, 1.0, A, 0, 1, n, 0, B, 0, 1, n, n * n,  # noqa
                                        0.0, C, 0, 1, n, n * n, n)
        line["cpu_baseline"] = cpu_baseline_obj(3 * 2.0 * n ** 4, lambda: [fn() for _ in range(3)],
                                                "3 C1 calls (batched_core, fp64)")
    emit(ctx, line)


# ----------------------------------------------------------------------------- small (configs[2])


def run_small(args, ctx):
    """configs[2]: batched GEMM C[mn[p]] = A[mk[p]] B[kn[p]], n = 8..64, P per
    GPU (default 10^6; weak: rank r holds batch range [r*P, (r+1)*P) of a
    global batch N*P).  HBM-bound: value reported with GB/s against HBM."""
    import torch
    from paper_1606_05696_b200 import _lib
    from paper_1606_05696_b200 import kernels as K
    dev = ctx.device
    dtype = torch.float32 if args.dtype == "f32" else torch.float64
    it = 4 if args.dtype == "f32" else 8
    hbm = load_peaks().get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"])
    tpeak, tnote = tensor_peak(args.dtype)
    P0 = args.batch
    head_n = 32
    sweep = []
    head = None
    for n in (8, 16, 32, 64):
        # fp64 n=64 at 10^6 entries would hold 98 GB: 2 x 10^5 (19.7 GB)
        P = min(P0, 200000) if (n == 64 and args.dtype == "f64") else P0
        a = torch.rand(n * n * P, dtype=dtype, device=dev)
        b = torch.rand(n * n * P, dtype=dtype, device=dev)
        c = torch.empty(n * n * P, dtype=dtype, device=dev)

        def f():
            K.strided_batched_gemm("N", "N", n, n, n, 1.0, a, n, n * n, b, n, n * n, 0.0, c, n,
                                   n * n, P)
        f()
        kernel = _lib.last_kernel()
        ms_l = event_ms(f, 5, dev)
        fl, nb = 2.0 * n ** 3 * P, 3.0 * n * n * P * it
        ent = {"n": n, "batch": P, "ms": round(ms_l, 4), "kernel": kernel,
               "gflops": round(fl / (ms_l * 1e-3) / 1e9, 1),
               "hbm_gbs": round(nb / (ms_l * 1e-3) / 1e9, 1),
               "frac_of_measured_hbm": round(nb / (ms_l * 1e-3) / 1e9 / hbm, 3)}
        if n == head_n:
            graph, lps = capture(f, dev)
            ms, clocks, launches = timed_steps(ctx, graph.replay, args.steps, args.warmup, lps)
            head = (n, P, fl, nb, ms, clocks, launches, kernel, ms_l)
        sweep.append(ent)
        del a, b, c
        torch.cuda.empty_cache()
    n, P, fl, nb, ms, clocks, launches, kernel, ms_l = head
    line = base_line(args, ctx, fl * ctx.world / (ms * 1e-3) / 1e9, ms, launches, clocks)
    line["config"] = {"workload": f"configs[2] batched GEMM n={n} (sweep n=8..64), P={P} per GPU",
                      "n": n, "batch_per_gpu": P, "global_batch": P * ctx.world,
                      "parallelism": f"dp{ctx.world}",
                      "sharding": f"weak: rank r holds batch range [r*{P}, (r+1)*{P}) of a global "
                                  f"batch {P * ctx.world} (no collective)",
                      "l2": f"operands {3 * nb / 3 / 1e9:.1f} GB > L2"}
    line["roofline"] = roofline_obj(fl, nb, ms_l, tpeak, tnote, hbm, kernel,
                                    f"{kernel}/small{n}/{args.dtype}")
    line["sweep"] = sweep
    line["hbm_gbs"] = round(nb / (ms * 1e-3) / 1e9, 1)
    if not args.no_e2e:
        Pe = P
        _, ha = pinned_np(n * n * Pe, dtype, seed=1)
        _, hb = pinned_np(n * n * Pe, dtype, seed=2)
        _, hc = pinned_np(n * n * Pe, dtype, fill=False)

        def host_call():
            K.strided_batched_gemm("N", "N", n, n, n, 1.0, ha, n, n * n, hb, n, n * n, 0.0, hc,
                                   n, n * n, Pe)
        host_call()
        reps = 3
        ctx.barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            host_call()
        dt = ctx.max_over_ranks(time.perf_counter() - t0) / reps
        line["e2e"] = {"value": round(2.0 * n ** 3 * Pe * ctx.world / dt / 1e9, 2),
                       "unit": "GFLOP/s", "h2d_bytes_per_step": 2 * n * n * Pe * it,
                       "d2h_bytes_per_step": n * n * Pe * it, "ms_per_step": round(dt * 1e3, 2),
                       "api": "kernels.strided_batched_gemm on pinned numpy buffers (host seam)"}
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        from oracle import cores
        Ps = 20000
        rng = np.random.default_rng(0)
        src = np.float32 if args.dtype == "f32" else np.float64
        A = rng.uniform(-1, 1, n * n * Ps).astype(src).astype(np.float64)
        B = rng.uniform(-1, 1, n * n * Ps).astype(src).astype(np.float64)
        C = np.empty(n * n * Ps)
        fn = lambda: cores.batched_core(n, n, n, 1.0, A, 0, 1, n, n * n, B, 0, 1, n, n * n,  # noqa
                                        0.0, C, 0, 1, n, n * n, Ps)
        line["cpu_baseline"] = cpu_baseline_obj(2.0 * n ** 3 * Ps, fn,
                                                f"n={n}, P={Ps} batched_core (fp64)")
    emit(ctx, line)


# ----------------------------------------------------------------------------- order4 (configs[4])


def run_order4(args, ctx):
    """configs[4]: C[mnpq] = A[mkp] B[nkq], n = 128 -- planned as a loop over p
    of a batched GEMM over q (reference planner), executed as ONE nested
    launch.  Weak: rank r holds the q-slab [r*n, (r+1)*n) of B and C; A is
    replicated (no collective)."""
    import torch
    from paper_1606_05696_b200 import _lib
    from paper_1606_05696_b200.layout import DenseTensor, Layout
    from paper_1606_05696_b200.notation import ContractionSpec
    from paper_1606_05696_b200.planner import execute_plan, plan_single_mode
    dev = ctx.device
    dtype = torch.float32 if args.dtype == "f32" else torch.float64
    it = 4 if args.dtype == "f32" else 8
    n = args.n if args.n != 256 else 128
    tpeak, tnote = tensor_peak(args.dtype)
    spec = ContractionSpec(tuple("mkp"), tuple("nkq"), tuple("mnpq"))
    la, lb, lc = Layout.packed((n,) * 3), Layout.packed((n,) * 3), Layout.packed((n,) * 4)
    g = torch.Generator(device=dev).manual_seed(7 + ctx.rank)
    a = DenseTensor(la, torch.rand(la.size, generator=g, dtype=dtype, device=dev) * 2 - 1)
    b = DenseTensor(lb, torch.rand(lb.size, generator=g, dtype=dtype, device=dev) * 2 - 1)
    c = DenseTensor(lc, torch.empty(lc.size, dtype=dtype, device=dev))
    plan = plan_single_mode(spec, la, lb, lc)
    f = lambda: execute_plan(plan, a, b, 1.0, 0.0, c)  # noqa: E731
    f()
    kernel = _lib.last_kernel()
    ms_l = event_ms(f, 5, dev)
    graph, lps = capture(f, dev)
    ms, clocks, launches = timed_steps(ctx, graph.replay, args.steps, args.warmup, lps)
    fl = 2.0 * n ** 5
    nb = it * (2 * n ** 3 + n ** 4)
    hbm = load_peaks().get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"])
    line = base_line(args, ctx, fl * ctx.world / (ms * 1e-3) / 1e9, ms, launches, clocks)
    line["config"] = {"workload": f"configs[4] C[mnpq]=A[mkp]B[nkq] n={n}",
                      "strategy": plan.strategy, "launches_per_contraction": lps,
                      "parallelism": f"dp{ctx.world}",
                      "sharding": shard_note(n, ctx.world, ctx.rank, "q (B's and C's last mode)"),
                      "l2": f"C = {it * n ** 4 / 1e9:.2f} GB > L2"}
    line["roofline"] = roofline_obj(fl, nb, ms_l, tpeak, tnote, hbm, kernel,
                                    f"{kernel}/order4/{args.dtype}")
    if not args.no_e2e:
        # the repo's public API with pinned host buffers: H2D of A and B, the
        # planned contraction, D2H of C
        pa, _ = pinned_np(la.size, dtype, seed=1)
        pb, _ = pinned_np(lb.size, dtype, seed=2)
        pc, _ = pinned_np(lc.size, dtype, fill=False)

        def e2e_step():
            a.data.copy_(pa, non_blocking=True)
            b.data.copy_(pb, non_blocking=True)
            f()
            pc.copy_(c.data, non_blocking=True)
            torch.cuda.synchronize()
        e2e_step()
        ctx.barrier()
        t0 = time.perf_counter()
        for _ in range(3):
            e2e_step()
        dt = ctx.max_over_ranks(time.perf_counter() - t0) / 3
        line["e2e"] = {"value": round(fl * ctx.world / dt / 1e9, 2), "unit": "GFLOP/s",
                       "h2d_bytes_per_step": it * (la.size + lb.size),
                       "d2h_bytes_per_step": it * lc.size, "ms_per_step": round(dt * 1e3, 2),
                       "api": "execute_plan on device DenseTensors, operands copied in from "
                              "pinned host memory and C copied out every step"}
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        from oracle import plan as oplan
        rng = np.random.default_rng(0)
        src = np.float32 if args.dtype == "f32" else np.float64
        A = rng.uniform(-1, 1, la.size).astype(src).astype(np.float64)
        B = rng.uniform(-1, 1, lb.size).astype(src).astype(np.float64)
        C = np.empty(lc.size)
        fn = lambda: oplan.contract(tuple("mkp"), tuple("nkq"), tuple("mnpq"),  # noqa: E731
                                    dict(m=n, n=n, p=n, k=n, q=n), A, B, 1.0, 0.0, C)
        line["cpu_baseline"] = cpu_baseline_obj(fl, fn, f"the full contraction at n={n} "
                                                "(planned loop of batched cores, fp64)",
                                                serial=False)
    emit(ctx, line)


# ----------------------------------------------------------------------------- hooi (configs[3])


def synthetic_tucker(n, r, device, dtype, seed=0, noise=1e-3):
    """Exact-rank Tucker tensor (core N(0,1), orthonormal factors from QR of
    N(0,1)) plus noise, column-major flat."""
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    core = torch.randn(r, r, r, device=device, generator=g, dtype=torch.float64)
    us = [torch.linalg.qr(torch.randn(n, r, device=device, generator=g,
                                      dtype=torch.float64))[0] for _ in range(3)]
    x = torch.einsum("ia,abc->ibc", us[0], core)
    x = torch.einsum("jb,ibc->ijc", us[1], x)
    x = torch.einsum("kc,ijc->ijk", us[2], x)
    x = x + noise * torch.randn(n, n, n, device=device, generator=g, dtype=torch.float64)
    return x.permute(2, 1, 0).contiguous().reshape(-1).to(dtype)


def hooi_flops(n, r):
    """Contraction FLOPs of one HOOI iteration with mode-0 reuse: chain(skip0)
    (two products), T x0, the two rank products of X0, the core."""
    return (2 * (n ** 3 * r + n * n * r * r) + 2 * n ** 3 * r + 2 * 2 * n * n * r * r
            + 2 * n * r ** 3)


def run_hooi(args, ctx):
    """configs[3]: HOOI of a synthetic 512^3 tensor, rank 32, fp32.  A step is
    one HOOI iteration; ms per iteration = difference of a (1+2K)- and a
    (1+K)-iteration run (both pay the HOSVD init, the graph capture and the
    final core), best of 3, each run timed with CUDA events on its stream."""
    import gc

    import torch
    import paper_1606_05696_b200 as sbt
    from paper_1606_05696_b200 import _lib
    from paper_1606_05696_b200.layout import DenseTensor, Layout
    dev = ctx.device
    dtype = torch.float32 if args.dtype == "f32" else torch.float64
    it = 4 if args.dtype == "f32" else 8
    n, r = (args.n if args.n != 256 else 512), 32
    if ctx.world > 1:
        return run_hooi_sharded(args, ctx, n, r, dtype)
    flat = synthetic_tucker(n, r, dev, dtype)
    t = DenseTensor(Layout.packed((n, n, n)), flat)
    sbt.hooi(t, (r, r, r), max_iters=1, tol=-1.0)  # warm-up: plans, libraries
    iters = max(2, args.steps)

    def run(k):
        gc.collect()   # Python's gen-2 GC passes (20-30 ms) must not land in a timed run
        gc.disable()
        try:
            torch.cuda.synchronize()
            n0 = _lib.launch_count()
            stream = torch.cuda.current_stream(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            m = sbt.hooi(t, (r, r, r), max_iters=k, tol=-1.0)
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) * 1e-3, m, _lib.launch_count() - n0
        finally:
            gc.enable()

    with ClockSampler(dev.index) as clocks:
        t_k = min(run(1 + iters)[0] for _ in range(3))
        runs = [run(1 + 2 * iters) for _ in range(3)]
    total, model, launches_long = min(runs, key=lambda x: x[0])
    per_iter = (total - t_k) / iters
    fl = hooi_flops(n, r)
    # HBM roofline of the iteration's mode products (algorithmic bytes, each
    # operand read and each product written once, mode-0 reuse)
    elems = 2 * n ** 3 + 5 * n * n * r + 4 * n * r * r + r ** 3
    nbytes = it * elems
    hbm = load_peaks().get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"])
    line = base_line(args, ctx, fl / per_iter / 1e9, per_iter * 1e3, None, clocks.summary())
    line["gpu_launches"] = launches_long
    line["gpu_launches_note"] = f"library launches of one {1 + 2 * iters}-iteration hooi() call"
    line["ms_per_iteration"] = round(per_iter * 1e3, 4)
    line["config"] = {"workload": f"configs[3] HOOI {n}^3 rank {r} {args.dtype}",
                      "iters_timed": iters, "hooi_paths": model.stats,
                      "contraction_gflop_per_iter": round(fl / 1e9, 2),
                      "fit_history": [round(f, 9) for f in model.fit_history],
                      "parallelism": "single GPU", "l2": f"T = {it * n ** 3 / 1e6:.0f} MB > L2"}
    line["roofline"] = {"bound": "hbm", "achieved": round(nbytes / per_iter / 1e9, 1),
                        "peak": hbm, "unit": "GB/s",
                        "frac": round(nbytes / (hbm * 1e9) / per_iter, 4),
                        "traffic": ncu_traffic(f"hooi_iteration/n{n}/{args.dtype}"),
                        "traffic_note": "ncu dram bytes of one iteration's launches "
                                        "(profiles/r02_ncu_hooi_iter.csv)",
                        "kernel": "HOOI iteration (CUDA graph)",
                        "algorithmic_bytes_per_iter": nbytes,
                        "floor_ms_per_iter": round(nbytes / (hbm * 1e9) * 1e3, 4),
                        "note": "bytes of the mode products only (T read twice, products "
                                "written once); the factor updates add latency, not bytes"}
    if not args.no_e2e:
        host, _ = pinned_np(n ** 3, dtype, fill=False)
        host.copy_(flat.cpu())
        k = 1 + iters

        def e2e_run():
            buf = torch.empty(n ** 3, dtype=dtype, device=dev)
            buf.copy_(host, non_blocking=True)
            m = sbt.hooi(DenseTensor(Layout.packed((n, n, n)), buf), (r, r, r), max_iters=k,
                         tol=-1.0)
            out = [m.core.data.cpu()] + [u.cpu() for u in m.factors]
            torch.cuda.synchronize()
            return out
        e2e_run()
        t0 = time.perf_counter()
        e2e_run()
        dt = time.perf_counter() - t0
        line["e2e"] = {"value": round(fl * k / dt / 1e9, 2), "unit": "GFLOP/s",
                       "h2d_bytes_per_step": it * n ** 3 // k,
                       "d2h_bytes_per_step": (it * r ** 3 + 8 * 3 * n * r) // k,
                       "ms_per_step": round(dt * 1e3 / k, 3),
                       "api": f"hooi() on a tensor copied from pinned host memory, {k} iterations "
                              "incl. HOSVD init and graph capture, core + factors copied back; "
                              "per-step = run / iterations"}
    if ctx.rank == 0 and not args.no_cpu:
        from oracle import tucker as otk
        xs = flat.cpu().numpy().astype(np.float64).reshape((n, n, n), order="F")
        cits = 2
        t0 = time.perf_counter()
        res = otk.hooi(xs, (r, r, r), max_iters=cits, tol=-1.0)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": round(fl * cits / dt / 1e9, 3), "unit": "GFLOP/s",
                                "cores": os.cpu_count(), "kind": "port",
                                "cpu_model": cpu_model(),
                                "sample": f"oracle/tucker.hooi {cits} iterations incl. HOSVD init "
                                          f"({dt:.1f} s; eigh for the reference's Jacobi)",
                                "fit_history": [round(f, 9) for f in res["fit_history"]]}
    emit(ctx, line)


def run_hooi_sharded(args, ctx, n, r, dtype):
    """HOOI with T slab-sharded along mode 2 (parallel.hooi_sharded): local
    products on the sm_100a kernels, NCCL all-reduce / all-gather per mode
    update.  Strong scaling (one T)."""
    import torch
    from paper_1606_05696_b200.parallel import hooi_sharded, slab
    dev = ctx.device
    from paper_1606_05696_b200.layout import DenseTensor, Layout
    flat = synthetic_tucker(n, r, dev, dtype)
    c0, c1 = slab(n, ctx.world, ctx.rank)
    # mode 2 is the slowest: the rank's slab is one contiguous chunk
    local = DenseTensor(Layout.packed((n, n, c1 - c0)), flat[c0 * n * n:c1 * n * n].clone())
    del flat
    hooi_sharded(local, (n, n, n), (r, r, r), max_iters=1, tol=-1.0)
    iters = max(2, args.steps)

    def run(k):
        torch.cuda.synchronize()
        ctx.barrier()
        torch.cuda.synchronize()
        stream = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = hooi_sharded(local, (n, n, n), (r, r, r), max_iters=k, tol=-1.0)
        e1.record(stream)
        torch.cuda.synchronize()
        return ctx.max_over_ranks(e0.elapsed_time(e1) * 1e-3), out

    with ClockSampler(dev.index) as clocks:
        t1 = min(run(1)[0] for _ in range(2))
        tk, out = run(1 + iters)
    per_iter = (tk - t1) / iters
    fl = hooi_flops(n, r)
    line = base_line(args, ctx, fl / per_iter / 1e9, per_iter * 1e3, None, clocks.summary())
    line["scaling"] = "strong"
    # roofline of the whole job: the products' algorithmic bytes (as for one GPU)
    # against the aggregate HBM bandwidth of the ranks
    it = 4 if dtype == torch.float32 else 8
    nbytes = it * (2 * n ** 3 + 5 * n * n * r + 4 * n * r * r + r ** 3)
    hbm = load_peaks().get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"]) * ctx.world
    line["roofline"] = {"bound": "hbm", "achieved": round(nbytes / per_iter / 1e9, 1),
                        "peak": hbm, "unit": "GB/s",
                        "frac": round(nbytes / (hbm * 1e9) / per_iter, 4), "traffic": None,
                        "kernel": "sharded HOOI iteration (all ranks)",
                        "note": f"aggregate HBM of {ctx.world} GPUs; the per-mode-update "
                                "collectives and the replicated factor updates are latency, "
                                "not bytes"}
    if not args.no_e2e:
        # end to end: every rank copies its slab in from pinned host memory and
        # brings the core and factors back
        host, _ = pinned_np(local.data.numel(), dtype, fill=False)
        host.copy_(local.data.cpu())
        k = 1 + iters

        def e2e_run():
            buf = torch.empty(local.data.numel(), dtype=dtype, device=dev)
            buf.copy_(host, non_blocking=True)
            core, us, _, _ = hooi_sharded(DenseTensor(local.layout, buf), (n, n, n), (r, r, r),
                                          max_iters=k, tol=-1.0)
            out = [core.cpu()] + [u.cpu() for u in us]
            torch.cuda.synchronize()
            return out
        e2e_run()
        ctx.barrier()
        t0 = time.perf_counter()
        e2e_run()
        dt = ctx.max_over_ranks(time.perf_counter() - t0)
        line["e2e"] = {"value": round(fl * k / dt / 1e9, 2), "unit": "GFLOP/s",
                       "h2d_bytes_per_step": it * local.data.numel() // k,
                       "d2h_bytes_per_step": (it * r ** 3 + 8 * 3 * n * r) // k,
                       "ms_per_step": round(dt * 1e3 / k, 3),
                       "api": f"parallel.hooi_sharded on slabs copied from pinned host memory, "
                              f"{k} iterations incl. the HOSVD init; core + factors copied "
                              "back; max over ranks"}
    line["config"] = {"workload": f"configs[3] HOOI {n}^3 rank {r} {args.dtype}",
                      "parallelism": f"T slab-sharded on mode 2 over {ctx.world} ranks "
                                     "(all-reduce / all-gather per mode update; HOSVD Gram of "
                                     "the sharded mode from ring-passed slabs, T never "
                                     "gathered; device-finished factor updates)",
                      "fit_history": [round(f, 9) for f in out[2]]}
    emit(ctx, line)


# ----------------------------------------------------------------------------- conventional


def run_conventional(args, ctx):
    """The paper's comparison (Fig. 1/4) on the device: every case as
    planned (transpose-free, one launch) vs conventional permute-then-GEMM
    (reference planner.py:411-465, policy "opt") vs batched GEMV."""
    import torch
    import paper_1606_05696_b200 as sbt
    from paper_1606_05696_b200.planner import execute_plan
    dtype = torch.float32 if args.dtype == "f32" else torch.float64
    n = args.n
    work = build_sets(case_shapes(n), n, dtype, ctx.device, 2, seed=7)
    per = {}
    tot_sb = tot_conv = tot_gemv = 0.0
    for cid, plan, a, b, c in work:
        conv = sbt.plan_conventional(plan.spec, a.layout, b.layout, c.layout, policy="opt")
        gv = sbt.plan_batched_gemv(plan.spec, a.layout, b.layout, c.layout)
        ms_sb = event_ms(lambda: execute_plan(plan, a, b, 1.0, 0.0, c), args.steps, ctx.device)
        ms_cv = event_ms(lambda: execute_plan(conv, a, b, 1.0, 0.0, c), args.steps, ctx.device)
        ms_gv = event_ms(lambda: execute_plan(gv, a, b, 1.0, 0.0, c), 2, ctx.device)
        tot_sb += ms_sb
        tot_conv += ms_cv
        tot_gemv += ms_gv
        per[cid] = {"sbgemm_ms": round(ms_sb, 4), "conventional_ms": round(ms_cv, 4),
                    "batched_gemv_ms": round(ms_gv, 4),
                    "transpositions": conv.predicted_transpositions,
                    "speedup": round(ms_cv / ms_sb, 2), "speedup_vs_gemv": round(ms_gv / ms_sb, 2)}
    fl = 2.0 * n ** 4 * len(work)
    line = {"metric": "transpose-free SBGEMM vs conventional permute+GEMM (36 cases); batched "
                      "GEMV as the third strategy",
            "value": round(tot_conv / tot_sb, 3), "unit": "x (conventional time / transpose-free "
                                                          "time)",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "dtype": args.dtype,
            "higher_is_better": True, "data": "synthetic",
            "config": {"workload": f"36-case sweep n={n} {args.dtype}, device, conventional "
                                   "policy opt",
                       "sbgemm_gflops": round(fl / (tot_sb * 1e-3) / 1e9, 1),
                       "conventional_gflops": round(fl / (tot_conv * 1e-3) / 1e9, 1),
                       "batched_gemv_gflops": round(fl / (tot_gemv * 1e-3) / 1e9, 1)},
            "per_case": per}
    emit(ctx, line)


# ----------------------------------------------------------------------------- output


def base_line(args, ctx, value, ms, launches, clocks):
    return {"metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ctx.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if args.dtype == "f64" else "f32 (3xTF32 tensor cores)",
            "data": "synthetic U[-1,1] operands (random init; no dataset), packed column-major",
            "config": {}, "roofline": None, "cpu_baseline": None, "e2e": None,
            "gpu_launches": launches, "clocks": clocks, "impl": "b200"}


def emit(ctx, line):
    if ctx.rank == 0:
        print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- reference arm


def run_reference(args):
    """The reference's algorithm on the host CPU (the oracle port: the
    reference numpy backend's planner lowering + numpy/OpenBLAS cores, fp64,
    all host threads) on this arm's config.  Under N ranks only rank 0 runs."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cores = os.cpu_count() or 1
    if args.config == "c1":
        from oracle import cores as oc
        n = 256
        rng = np.random.default_rng(0)
        A, B = rng.uniform(-1, 1, n * n), rng.uniform(-1, 1, n ** 3)
        C = np.empty(n ** 3)
        fn = lambda: oc.batched_core(n, n, n, 1.0, A, 0, 1, n, 0, B, 0, 1, n, n * n,  # noqa
                                     0.0, C, 0, 1, n, n * n, n)
        flops, sample, workload = 2.0 * n ** 4, "one C1 call per step (batched_core)", \
            "configs[0] C1 strided_batched_gemm n=256"
    else:
        n = args.n
        fn, flops, nc = cpu_sweep(n, args.dtype)
        sample = f"all {nc} cases at n={n} per step"
        workload = f"36-case single-index sweep (configs[1]) at n={n}"
    for _ in range(max(1, args.warmup)):
        fn()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    ms = statistics.median(times) * 1e3
    value = flops / (ms * 1e-3) / 1e9
    out = {"metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": args.dtype, "data": "synthetic U[-1,1]",
           "config": {"workload": workload, "n": n}, "impl": "reference",
           "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": cores,
                            "kind": "port", "cpu_model": cpu_model(),
                            "sample": f"{sample} (oracle port of the reference planner + "
                                      "numpy/OpenBLAS cores, fp64, all host threads)"},
           "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--dtype", choices=("f32", "f64"), default=None)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--config", choices=("sweep", "c1", "small", "order4", "hooi",
                                         "conventional"), default="sweep")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-group", action="store_true",
                    help="sweep: issue the cases as separate calls instead of one grouped call")
    ap.add_argument("--batch", type=int, default=1000000)
    args = ap.parse_args()
    if args.dtype is None:
        args.dtype = DEFAULT_DTYPE[args.config]
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args)
        return
    ctx = Ctx()
    try:
        {"sweep": run_sweep, "c1": run_c1, "small": run_small, "order4": run_order4,
         "hooi": run_hooi, "conventional": run_conventional}[args.config](args, ctx)
    finally:
        ctx.close()


if __name__ == "__main__":
    main()
