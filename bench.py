#!/usr/bin/env python
"""Benchmark: single-index contraction throughput on B200 (BASELINE.json configs[1]).

A step is the sweep of all 36 second-order x third-order single-index
contraction cases (flat GEMM / strided batched / exceptional) at extent n
(default n=256, fp32 via 3xTF32 tensor cores), each planned by the reference's
dispatcher semantics and executed as one launch of the sm_100a library.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n 256] [--dtype f32|f64]
    python bench.py --impl reference ...   # the reference algorithm on the host CPU

Weak scaling: every rank runs the full per-GPU sweep on its own operands (the
batch/free-mode shard of a problem N times larger); there is no data-path
collective.  value = FLOPs of all ranks / max-over-ranks device time.
Inputs: 4 (or a multiple of the stream count) rotating operand sets per step,
each larger than L2 at n >= 256, so consecutive cases never hit L2 for their
operands; below n = 256 the working set fits L2 and the config line says so.
"""
from __future__ import annotations

import argparse
import json
import os
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


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["source"] = "measured"
        return d
    return dict(FALLBACK_PEAKS)


def case_shapes(n):
    from paper_1606_05696_b200.planner import enumerate_cases
    out = []
    for case in enumerate_cases(2, 3):
        ext = dict(m=n, n=n, p=n, k=n)
        out.append((case, ext))
    return out


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


# ----------------------------------------------------------------------------- GPU arm


def build_sets(cases, n, dtype, device, nsets, seed, distinct_c=False):
    import torch
    from paper_1606_05696_b200.layout import DenseTensor, Layout
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
        spec_labels = (case.labels_a, case.labels_b, case.labels_c)
        la = Layout.packed([ext[l] for l in case.labels_a])
        lb = Layout.packed([ext[l] for l in case.labels_b])
        lc = Layout.packed([ext[l] for l in case.labels_c])
        from paper_1606_05696_b200.notation import ContractionSpec
        plan = plan_single_mode(ContractionSpec(*spec_labels), la, lb, lc)
        a, b, c = sets[i % nsets]
        if distinct_c:  # grouped execution: every case writes its own C
            c = torch.empty(size_b, device=device, dtype=dtype)
        # the order-2 operand may be A or B of the case: bind buffers by size
        ta = DenseTensor(la, a if la.size == size_a else b)
        tb = DenseTensor(lb, a if lb.size == size_a else b)
        work.append((case.case_id, plan, ta, tb, DenseTensor(lc, c)))
    return work


def ncu_traffic(kernel, n, dtype):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel from the committed ncu --set full capture (profiles/ncu_traffic.json),
    or None when no capture of this (kernel, n, dtype) exists."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        table = json.loads(p.read_text())
    except ValueError:
        return None
    return table.get(f"{kernel}/n{n}/{dtype}")


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_1606_05696_b200 import _lib
    from paper_1606_05696_b200.planner import execute_plan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(device)
    dtype = torch.float32 if args.dtype == "f32" else torch.float64
    itemsize = 4 if dtype == torch.float32 else 8
    n = args.n
    sustained = None
    tf32_burst = None
    if dtype == torch.float32:
        try:  # before any heavy work: burst = clocks at max
            tf32_burst = _lib.probe_tf32_peak()
        except Exception:
            tf32_burst = None
    cases = case_shapes(n)
    # 4 rotating operand sets: with the step's cases issued round-robin on 2
    # streams, cases that can run concurrently never share a buffer (cases
    # sharing a set share a stream and are ordered)
    # grouped mode: the step's independent contractions go through ONE
    # execute_plans call (one persistent launch per kernel configuration);
    # every case then needs its own C (36 x n^3 elements)
    # (n >= 512: one case is >= 0.5 ms, launch overheads are negligible and
    # separate launches on two streams fill each other's tails better)
    # (n <= 64: almost nothing is pair-groupable and every case is ~1 us of
    # work; execute_plans forks such calls over internal streams, so the step
    # still overlaps its launches: 2x a single-stream issue, measured)
    group = (not args.no_group) and n <= 256
    if args.streams is None:
        args.streams = 2
    # operand sets: a multiple of the stream count, so cases on different
    # streams never share a buffer
    nsets = 4 * ((args.streams + 3) // 4) if args.streams > 4 else 4
    work = build_sets(cases, n, dtype, device, nsets, seed=1234 + rank, distinct_c=group)
    from paper_1606_05696_b200.planner import execute_plans
    exceptional = {cid for cid, *_ in work if cid in EXCEPTIONAL_CASES}
    stream = torch.cuda.current_stream(device)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[device.index])

    nc = len(work)
    kernel_of = {}
    for cid, plan, a, b, c in work:  # one untimed pass to learn kernel families
        execute_plan(plan, a, b, 1.0, 0.0, c)
        kernel_of[cid] = _lib.last_kernel()
    for _ in range(args.warmup):
        for cid, plan, a, b, c in work:
            execute_plan(plan, a, b, 1.0, 0.0, c)
    # (1) per-case attribution: events between the launches, no graph
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nc + 1)]
          for _ in range(args.steps)]
    torch.cuda.synchronize()
    for st in range(args.steps):
        ev[st][0].record(stream)
        for i, (cid, plan, a, b, c) in enumerate(work):
            execute_plan(plan, a, b, 1.0, 0.0, c)
            ev[st][i + 1].record(stream)
    torch.cuda.synchronize()
    per_case = [[ev[st][i].elapsed_time(ev[st][i + 1]) for st in range(args.steps)]
                for i in range(nc)]
    nograph_ms = ev[0][0].elapsed_time(ev[-1][nc]) / args.steps
    group_attr = None
    if group:
        # one grouped launch per subset (plain cases / exceptional cases), each
        # captured in a CUDA graph and timed with events on the launching stream
        subsets = {"tc_tf32x3_pair_group" if dtype == torch.float32 else "grouped_f64":
                   [w for w in work if w[0] not in exceptional],
                   "tc_tf32x3_pair_group_bb" if dtype == torch.float32 else "grouped_f64_bb":
                   [w for w in work if w[0] in exceptional]}
        group_attr = {}
        for name, sub in subsets.items():
            if not sub:
                continue
            calls = [(plan, a, b, 1.0, 0.0, c) for cid, plan, a, b, c in sub]
            for _ in range(2):
                execute_plans(calls)
            sub_graph = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(device)
            cap.wait_stream(stream)
            with torch.cuda.stream(cap):
                with torch.cuda.graph(sub_graph, stream=cap):
                    execute_plans(calls)
            stream.wait_stream(cap)
            sub_graph.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(args.steps):
                sub_graph.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            group_attr[name] = {"cases": len(sub), "ms": round(ms, 4),
                                "launch_kernel": _lib.last_kernel(),
                                "tflops": round(len(sub) * 2.0 * n ** 4 / (ms * 1e-3) / 1e12, 2)}

    # (2) the timed steps: the step's 36 independent contractions issued
    # round-robin on args.streams CUDA streams (one library launch each, so a
    # kernel's tail overlaps the next one's start), captured once into a CUDA
    # graph (no host launch gaps) and replayed K times
    side = [torch.cuda.Stream(device) for _ in range(max(0, args.streams - 1))]

    def issue_step(main):
        if group:
            # the step's 36 independent contractions as ONE execute_plans call:
            # the library runs each kernel configuration as one persistent launch
            # (plain / exceptional) on its own internal stream and forks the
            # remaining calls, joining back to this stream
            with torch.cuda.stream(main):
                execute_plans([(plan, a, b, 1.0, 0.0, c) for cid, plan, a, b, c in work])
            return
        for sd in side:
            sd.wait_stream(main)
        lanes = [main] + side
        for i, (cid, plan, a, b, c) in enumerate(work):
            with torch.cuda.stream(lanes[i % len(lanes)]):
                execute_plan(plan, a, b, 1.0, 0.0, c)
        for sd in side:
            main.wait_stream(sd)

    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device)
        cap.wait_stream(stream)
        cap_launch0 = _lib.launch_count()
        with torch.cuda.stream(cap):
            with torch.cuda.graph(graph, stream=cap):
                issue_step(cap)
        launches_per_step = _lib.launch_count() - cap_launch0
        stream.wait_stream(cap)
        for _ in range(args.warmup):
            graph.replay()
    t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    with ClockSampler(device.index) as clocks:
        time.sleep(0.05)  # sampler running before the timed region starts
        t0e.record(stream)
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                issue_step(stream)
        t1e.record(stream)
        torch.cuda.synchronize()
    launches = ((_lib.launch_count() - launches0) if graph is None
                else launches_per_step * args.steps)
    barrier()
    total_ms = t0e.elapsed_time(t1e)
    kern_ms = sum(sum(x) for x in per_case)
    t = torch.tensor([total_ms], device=device, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps

    fl, by = flops_bytes(n, itemsize)
    step_flops = fl * nc
    value = step_flops * world / (ms_per_step * 1e-3) / 1e9

    peaks = load_peaks()
    if dtype == torch.float32:
        try:
            if tf32_burst is None:
                raise RuntimeError("tf32 probe failed")
            peak_tflops = tf32_burst / 3.0
            peak_note = (f"3xTF32 = measured tcgen05 kind::tf32 dense peak {tf32_burst:.0f} "
                         "TFLOP/s / 3 (sbt_probe_tf32_peak, random operands, in-run before the "
                         "timed work: burst)")
            if args.sustained_probe or n >= 512:
                sustained = _lib.probe_tf32_sustained(3.0) / 3.0
                # n >= 512: the per-case pass runs for hundreds of ms under the
                # power cap, so the sustained figure is the denominator
                peak_tflops = sustained
                peak_note += (f"; frac uses the sustained peak {3 * sustained:.0f} TFLOP/s / 3 "
                              "(3 s back to back: the power-capped clock)")
        except Exception:
            peak_tflops = peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"]) / 2.0 / 3.0
            peak_note = f"3xTF32 = bf16_tflops({peaks['source']})/2/3 (tf32 probe failed)"
    else:
        try:
            peak_tflops = _lib.probe_fp64_peak("dmma")
            peak_note = "fp64 DMMA measured in-run by sbt_probe_fp64_peak"
        except Exception:
            peak_tflops = FP64_NOMINAL_TFLOPS
            peak_note = "fp64 DMMA nominal (datasheet 37 TFLOP/s)"
    hbm = peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"])
    roof_ms = max(fl / (peak_tflops * 1e12), by / (hbm * 1e9)) * 1e3 * nc
    # dominant kernel family
    fam_ms, fam_flops = {}, {}
    for i, (cid, *_r) in enumerate(work):
        k = kernel_of[cid]
        fam_ms[k] = fam_ms.get(k, 0.0) + statistics.mean(per_case[i])
        fam_flops[k] = fam_flops.get(k, 0.0) + fl
    if group_attr:
        fam_ms = {k: v["ms"] for k, v in group_attr.items()}
        fam_flops = {k: v["cases"] * fl for k, v in group_attr.items()}
        kern_ms = sum(fam_ms.values()) * args.steps
    dom = max(fam_ms, key=fam_ms.get)
    dom_tflops = fam_flops[dom] / (fam_ms[dom] * 1e-3) / 1e12
    bound = "tensor" if fl / by > (peak_tflops * 1e12) / (hbm * 1e9) else "hbm"
    dom_gbs = (fam_flops[dom] / fl) * by / (fam_ms[dom] * 1e-3) / 1e9
    achieved = dom_tflops if bound == "tensor" else dom_gbs
    peak = peak_tflops if bound == "tensor" else hbm
    roofline = {
        "bound": bound, "kernel": dom, "unit": "TFLOP/s" if bound == "tensor" else "GB/s",
        "achieved": round(achieved, 3), "peak": round(peak, 2),
        "frac": round(achieved / peak, 4),
        "traffic": ncu_traffic(dom, n, args.dtype), "peak_source": peak_note,
        "hbm_peak_gbs": hbm, "hbm_achieved_gbs": round(dom_gbs, 1),
        "peak_burst": round(tf32_burst / 3.0, 2) if tf32_burst else None,
        "peak_sustained": round(sustained, 2) if sustained else None,
        "algorithmic": {"flop_per_case": fl, "bytes_per_case": by,
                        "note": "per case (one launch): 2n^4 FLOP; s*(n^2 + 2n^3) B (A read, "
                                "B read, C written once; beta = 0)"},
        "step_frac_of_roofline": round(roof_ms / ms_per_step, 4),
        "kernel_share_of_step": round(fam_ms[dom] / (kern_ms / args.steps), 4),
        "measured_in": ("CUDA events on the launching stream around each grouped launch "
                        "(plain cases / exceptional cases)" if group_attr else
                        "CUDA events on the launching stream, per-case pass without graph"),
        "per_launch_cases": (group_attr[dom]["cases"] if group_attr else 1),
    }
    per_case_out = {work[i][0]: {"ms": round(statistics.median(per_case[i]), 4),
                                 "kernel": kernel_of[work[i][0]],
                                 "tflops": round(fl / (statistics.median(per_case[i]) * 1e-3)
                                                 / 1e12, 2)}
                    for i in range(nc)}

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, work, device, dtype, itemsize, n, step_flops, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(n, args)

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32(3xTF32)" if dtype == torch.float32 else "f64",
            "data": "synthetic U[-1,1] operands, packed column-major",
            "config": {"workload": f"36-case single-index sweep (configs[1]) at n={n}",
                       "n": n, "cases": nc, "gflop_per_step_per_gpu": round(step_flops / 1e9, 2),
                       "parallelism": f"batch-sharded x{world} (no collective)",
                       "l2": (f"{nsets} rotating operand sets, each > L2 (126 MB)" if n >= 256 else
                              f"{nsets} rotating operand sets; at n={n} the working set fits "
                              "L2, so inputs are L2-warm (no flush between steps)"),
                       "issue": ("one execute_plans call per step: the 36 independent "
                                 "contractions as grouped persistent launches (plain / "
                                 "exceptional)" if group else
                                 f"36 independent launches per step, round-robin on "
                                 f"{args.streams} stream(s)"),
                       "alpha": 1.0, "beta": 0.0},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "cuda_graph": graph is not None, "streams": args.streams,
            "grouped": group, "group_launches": group_attr,
            "ms_per_step_nograph": round(nograph_ms, 4),
            "clocks": clocks.summary(),
            "wall_ms_timed_region": round(total_ms, 3),
            "per_case": per_case_out,
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, work, device, dtype, itemsize, n, step_flops, world):
    """Same sweep through the public API with host buffers.  Every step: copy
    the step's two operands (the order-2 and order-3 tensors all 36 cases
    contract, as in the CPU arm) from pinned host memory, run the 36 planned
    contractions, and copy every case's C back to pinned host memory.  The
    device->host copies run on a second stream (their own copy engine) and
    overlap the next cases' compute; two device C buffers rotate, each reused
    only after its copy-out finished.  Timed on the host around whole steps
    (one device sync per step)."""
    import torch
    from paper_1606_05696_b200.layout import DenseTensor
    from paper_1606_05696_b200.planner import execute_plan
    size_a, size_b = n * n, n ** 3
    ha = torch.empty(size_a, dtype=dtype).uniform_(-1, 1).pin_memory()
    hb = torch.empty(size_b, dtype=dtype).uniform_(-1, 1).pin_memory()
    hc = [torch.empty(size_b, dtype=dtype).pin_memory() for _ in range(2)]
    da = torch.empty(size_a, dtype=dtype, device=device)
    db = torch.empty(size_b, dtype=dtype, device=device)
    dc = [torch.empty(size_b, dtype=dtype, device=device) for _ in range(2)]
    jobs = []
    for i, (cid, plan, a, b, c) in enumerate(work):
        ta = DenseTensor(a.layout, da if a.layout.size == size_a else db)
        tb = DenseTensor(b.layout, da if b.layout.size == size_a else db)
        jobs.append((plan, ta, tb, [DenseTensor(c.layout, x) for x in dc]))
    s_comp = torch.cuda.Stream(device)
    s_out = torch.cuda.Stream(device)
    copied = [torch.cuda.Event() for _ in range(2)]
    for e in copied:
        e.record(s_out)

    def step():
        with torch.cuda.stream(s_comp):
            da.copy_(ha, non_blocking=True)
            db.copy_(hb, non_blocking=True)
            for i, (plan, ta, tb, tcs) in enumerate(jobs):
                j = i % 2
                s_comp.wait_event(copied[j])          # C buffer j drained to the host
                execute_plan(plan, ta, tb, 1.0, 0.0, tcs[j])
                done = torch.cuda.Event()
                done.record(s_comp)
                s_out.wait_event(done)
                with torch.cuda.stream(s_out):
                    hc[j].copy_(dc[j], non_blocking=True)
                copied[j].record(s_out)
        torch.cuda.synchronize(device)

    step()
    steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    h2d = itemsize * (size_a + size_b)
    d2h = len(jobs) * itemsize * size_b
    return {"value": round(step_flops * world / dt / 1e9, 2), "unit": "GFLOP/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": round(dt * 1e3, 3), "steps": steps,
            "api": "paper_1606_05696_b200.execute_plan; operands copied in from pinned host "
                   "memory once per step, every case's C copied out (overlapped on a 2nd stream)"}


# ----------------------------------------------------------------------------- other configs


def _time_steps(fn, steps, warmup):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def run_config(args):
    """BASELINE configs[2..4] as single-GPU measurements (one JSON line each):
    small   -- batched GEMM n=8/16/32/64, P=10^6 (HBM-bound; GB/s vs measured copy BW)
    order4  -- C[mnpq] = A[mkp] B[nkq], n=128: one nested-batched launch
    hooi    -- Tucker HOOI 512^3 rank 32 fp32: ms per iteration, contraction GFLOP/s"""
    import torch
    from paper_1606_05696_b200 import _lib, kernels
    from paper_1606_05696_b200.layout import DenseTensor, Layout
    from paper_1606_05696_b200.notation import ContractionSpec
    from paper_1606_05696_b200.planner import execute_plan, plan_single_mode
    torch.cuda.set_device(0)
    dtype = torch.float32 if args.dtype == "f32" else torch.float64
    it = 4 if dtype == torch.float32 else 8
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"])
    out = []
    if args.config == "small":
        P0 = args.batch
        for n in (8, 16, 32, 64):
            # fp64 n=64 at 10^6 entries would hold 98 GB: run 2 x 10^5 (19.7 GB)
            P = min(P0, 200000) if (n == 64 and dtype == torch.float64) else P0
            a = torch.rand(n * n * P, dtype=dtype, device="cuda")
            b = torch.rand(n * n * P, dtype=dtype, device="cuda")
            c = torch.empty(n * n * P, dtype=dtype, device="cuda")
            f = lambda: kernels.strided_batched_gemm("N", "N", n, n, n, 1.0, a, n, n * n, b, n,  # noqa: E731
                                                     n * n, 0.0, c, n, n * n, P)
            ms = _time_steps(f, args.steps, args.warmup)
            gbs = 3 * n * n * P * it / (ms * 1e-3) / 1e9
            out.append({"n": n, "batch": P, "ms": round(ms, 4), "kernel": _lib.last_kernel(),
                        "gflops": round(2 * n ** 3 * P / (ms * 1e-3) / 1e9, 1),
                        "hbm_gbs": round(gbs, 1), "frac_of_measured_hbm": round(gbs / hbm, 3)})
            del a, b, c
        value = out[2]["hbm_gbs"] if len(out) > 2 else out[-1]["hbm_gbs"]
        line = {"metric": "batched small-matrix GEMM HBM throughput (n=32 headline)",
                "value": value, "unit": "GB/s", "roofline": {
                    "bound": "hbm", "achieved": value, "peak": hbm, "unit": "GB/s",
                    "frac": round(value / hbm, 3), "traffic": None},
                "config": {"workload": f"configs[2] batched GEMM, P={P0}"}, "sweep": out}
    elif args.config == "order4":
        n = args.n if args.n != 256 else 128
        spec = ContractionSpec(tuple("mkp"), tuple("nkq"), tuple("mnpq"))
        la, lb, lc = Layout.packed((n,) * 3), Layout.packed((n,) * 3), Layout.packed((n,) * 4)
        a = DenseTensor(la, torch.rand(la.size, dtype=dtype, device="cuda"))
        b = DenseTensor(lb, torch.rand(lb.size, dtype=dtype, device="cuda"))
        c = DenseTensor(lc, torch.empty(lc.size, dtype=dtype, device="cuda"))
        plan = plan_single_mode(spec, la, lb, lc)
        n0 = _lib.launch_count()
        execute_plan(plan, a, b, 1.0, 0.0, c)
        launches = _lib.launch_count() - n0
        ms = _time_steps(lambda: execute_plan(plan, a, b, 1.0, 0.0, c), args.steps, args.warmup)
        flops = 2.0 * n ** 5
        kernel = _lib.last_kernel()
        # roofline: the slower of the tensor pipe at its measured peak (3xTF32 =
        # TF32 probe / 3; fp64 DMMA probe) and the operand + C bytes at HBM rate
        if dtype == torch.float32:
            tpeak, tsrc = _lib.probe_tf32_peak() / 3.0, "3xTF32 = measured tcgen05 TF32 / 3"
        else:
            tpeak, tsrc = _lib.probe_fp64_peak("dmma"), "measured DMMA"
        nbytes = it * (2 * n ** 3 + n ** 4)
        t_floor = max(flops / (tpeak * 1e12), nbytes / (hbm * 1e9)) * 1e3
        line = {"metric": "4th-order contraction GFLOP/s", "value": round(flops / (ms * 1e-3) / 1e9, 1),
                "unit": "GFLOP/s", "ms_per_step": round(ms, 4),
                "roofline": {"bound": "tensor" if flops / tpeak / 1e12 > nbytes / hbm / 1e9 else "hbm",
                             "achieved": round(flops / (ms * 1e-3) / 1e12, 2), "peak": round(tpeak, 2),
                             "unit": "TFLOP/s", "frac": round(t_floor / ms, 3), "traffic": None,
                             "peak_source": tsrc, "hbm_peak_gbs": hbm,
                             "algorithmic_bytes": nbytes,
                             "note": "frac = max(flop / tensor peak, bytes / HBM) / measured time"},
                "config": {"workload": f"configs[4] C[mnpq]=A[mkp]B[nkq] n={n}",
                           "strategy": plan.strategy, "launches_per_contraction": launches,
                           "kernel": kernel}}
    elif args.config == "hooi":
        import paper_1606_05696_b200 as sbt
        n, r = (args.n if args.n != 256 else 512), 32
        g = torch.Generator(device="cuda").manual_seed(0)
        core = torch.randn(r, r, r, device="cuda", generator=g, dtype=torch.float64)
        us = [torch.linalg.qr(torch.randn(n, r, device="cuda", generator=g,
                                          dtype=torch.float64))[0] for _ in range(3)]
        x = torch.einsum("ia,abc->ibc", us[0], core)
        x = torch.einsum("jb,ibc->ijc", us[1], x)
        x = torch.einsum("kc,ijc->ijk", us[2], x)
        x = x + 1e-3 * torch.randn(n, n, n, device="cuda", generator=g, dtype=torch.float64)
        t = DenseTensor(Layout.packed((n, n, n)), x.permute(2, 1, 0).contiguous().reshape(-1).to(dtype))
        del x
        sbt.hooi(t, (r, r, r), max_iters=1, tol=-1.0)  # warm-up: plans, libraries
        iters = max(2, args.steps)

        import gc

        def run(k):
            # Python's cyclic GC (20-30 ms gen-2 passes in this process) would
            # land at random inside timed runs: collect first, pause it inside
            gc.collect()
            gc.disable()
            try:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                m = sbt.hooi(t, (r, r, r), max_iters=k, tol=-1.0)
                torch.cuda.synchronize()
                return time.perf_counter() - t0, m
            finally:
                gc.enable()

        # steady-state cost per iteration = difference of a (1+K)- and a
        # (1+2K)-iteration run (both include the HOSVD init, the one-time
        # capture of the iteration graph and the final core); best of 3 each.
        # The 1-iteration run gives the per-iteration cost including capture.
        t_init = min(run(1)[0] for _ in range(3))
        t_k = min(run(1 + iters)[0] for _ in range(3))
        runs = [run(1 + 2 * iters) for _ in range(3)]
        total, model = min(runs, key=lambda x: x[0])
        per_iter = (total - t_k) / iters
        per_iter_first_k = (t_k - t_init) / iters
        # contraction FLOPs per iteration with mode-0 reuse: chain(skip0) 2 products,
        # T x0, two 32-rank products, core
        fl = 2 * (n ** 3 * r + n * n * r * r) + 2 * n ** 3 * r + 2 * 2 * n * n * r * r + 2 * n * r ** 3
        line = {"metric": "Tucker HOOI ms per iteration", "value": round(per_iter * 1e3, 3),
                "unit": "ms", "higher_is_better": False,
                "config": {"workload": f"configs[3] HOOI {n}^3 rank {r} {args.dtype}",
                           "init_plus_one_iter_ms": round(t_init * 1e3, 1),
                           "ms_per_iter_incl_graph_capture": round(per_iter_first_k * 1e3, 3),
                           "iters_timed": iters,
                           "hooi_paths": model.stats,
                           "contraction_gflop_per_iter": round(fl / 1e9, 2),
                           "fit_history": [round(f, 8) for f in model.fit_history]}}
        # HBM roofline of the iteration's mode products (algorithmic bytes, each
        # operand read and each product written once, mode-0 reuse): T twice,
        # five n^2 r-sized tensors, four n r^2, the r^3 core
        elems = 2 * n ** 3 + 5 * n * n * r + 4 * n * r * r + r ** 3
        nbytes = it * elems
        floor_ms = nbytes / (hbm * 1e9) * 1e3
        line["roofline"] = {"bound": "hbm", "achieved": round(nbytes / per_iter / 1e9, 1),
                            "peak": hbm, "unit": "GB/s",
                            "frac": round(floor_ms / (per_iter * 1e3), 3), "traffic": None,
                            "algorithmic_bytes_per_iter": nbytes,
                            "floor_ms_per_iter": round(floor_ms, 4),
                            "note": "bytes of the mode products only; the factor updates "
                                    "(skinny fp64 products, Ritz kernels) add latency, "
                                    "not bytes"}
    elif args.config == "conventional":
        # the paper's comparison (Fig. 1/4) on the device: every case
        # as planned (transpose-free, one launch) vs conventional
        # permute-then-GEMM (reference planner.py:411-465, policy "opt")
        import paper_1606_05696_b200 as sbt
        n = args.n
        cases = case_shapes(n)
        work = build_sets(cases, n, dtype, "cuda", 2, seed=7)
        per = {}
        tot_sb = tot_conv = 0.0
        tot_gemv = 0.0
        for cid, plan, a, b, c in work:
            conv = sbt.plan_conventional(plan.spec, a.layout, b.layout, c.layout, policy="opt")
            gv = sbt.plan_batched_gemv(plan.spec, a.layout, b.layout, c.layout)
            ms_sb = _time_steps(lambda: execute_plan(plan, a, b, 1.0, 0.0, c), args.steps,
                                args.warmup)
            ms_cv = _time_steps(lambda: execute_plan(conv, a, b, 1.0, 0.0, c), args.steps,
                                args.warmup)
            ms_gv = _time_steps(lambda: execute_plan(gv, a, b, 1.0, 0.0, c), max(1, args.steps // 2),
                                1)
            tot_sb += ms_sb
            tot_conv += ms_cv
            tot_gemv += ms_gv
            per[cid] = {"sbgemm_ms": round(ms_sb, 4), "conventional_ms": round(ms_cv, 4),
                        "batched_gemv_ms": round(ms_gv, 4),
                        "transpositions": conv.predicted_transpositions,
                        "speedup": round(ms_cv / ms_sb, 2),
                        "speedup_vs_gemv": round(ms_gv / ms_sb, 2)}
        fl = 2.0 * n ** 4 * len(work)
        line = {"metric": "transpose-free SBGEMM vs conventional permute+GEMM (36 cases); "
                          "batched GEMV as the third strategy",
                "value": round(tot_conv / tot_sb, 3), "unit": "x (conventional time / "
                "transpose-free time)",
                "config": {"workload": f"36-case sweep n={n} {args.dtype}, device, "
                                       "conventional policy opt",
                           "sbgemm_gflops": round(fl / (tot_sb * 1e-3) / 1e9, 1),
                           "conventional_gflops": round(fl / (tot_conv * 1e-3) / 1e9, 1),
                           "batched_gemv_gflops": round(fl / (tot_gemv * 1e-3) / 1e9, 1)},
                "per_case": per}
    else:
        raise SystemExit(f"unknown config {args.config}")
    line.update({"n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                 "dtype": args.dtype, "data": "synthetic"})
    line.setdefault("higher_is_better", True)
    print(json.dumps(line))


# ----------------------------------------------------------------------------- CPU arm


# bounded per-step sample for --impl reference: one case of every dispatch class
REFERENCE_SAMPLE = ("1.1", "1.3", "2.4", "3.4", "5.5", "6.4")


def cpu_sample(n, dtype_name, only=None):
    """The reference algorithm (oracle port: planner lowering + numpy/OpenBLAS
    cores, fp64 arithmetic as the reference) on the same 36-case sweep."""
    from oracle import plan as oplan
    from paper_1606_05696_b200.planner import enumerate_cases  # case catalogue only
    rng = np.random.default_rng(0)
    src_dtype = np.float32 if dtype_name == "f32" else np.float64
    a = rng.uniform(-1, 1, n * n).astype(src_dtype).astype(np.float64)
    b = rng.uniform(-1, 1, n ** 3).astype(src_dtype).astype(np.float64)
    c = np.empty(n ** 3)
    cases = [c for c in enumerate_cases(2, 3) if only is None or c.case_id in only]
    t0 = time.perf_counter()
    for case in cases:
        ext = dict(m=n, n=n, p=n, k=n)
        x = a if len(case.labels_a) == 2 else b
        y = a if len(case.labels_b) == 2 else b
        oplan.contract(case.labels_a, case.labels_b, case.labels_c, ext, x, y, 1.0, 0.0, c)
    dt = time.perf_counter() - t0
    return len(cases) * 2.0 * n ** 4 / dt / 1e9, dt, len(cases)


def cpu_baseline(n, args):
    cores = os.cpu_count() or 1
    gflops, dt, ncases = cpu_sample(n, args.dtype)
    return {"value": round(gflops, 3), "unit": "GFLOP/s", "cores": cores, "kind": "port",
            "sample": f"all {ncases} cases at n={n}, fp64 arithmetic on "
                      f"{'fp32-rounded ' if args.dtype == 'f32' else ''}inputs, "
                      f"numpy/OpenBLAS ({dt:.1f} s)"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    n = args.n
    cpu_sample(min(n, 64), args.dtype, REFERENCE_SAMPLE)  # warm-up (BLAS threads, caches)
    times = []
    ncases = 0
    for _ in range(args.steps):
        gflops, dt, ncases = cpu_sample(n, args.dtype, REFERENCE_SAMPLE)
        times.append(dt)
    ms = statistics.median(times) * 1e3
    value = ncases * 2.0 * n ** 4 / (ms * 1e-3) / 1e9
    out = {"metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic U[-1,1]",
           "config": {"workload": f"36-case single-index sweep (configs[1]) at n={n}", "n": n,
                      "cases_timed_per_step": ncases},
           "impl": "reference",
           "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": cores,
                            "kind": "port",
                            "sample": f"{ncases} of the 36 cases ({', '.join(REFERENCE_SAMPLE)}) at "
                                      f"n={n} per step (oracle port of the reference planner + "
                                      "numpy/OpenBLAS cores, all host threads)"},
           "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--dtype", choices=("f32", "f64"), default="f32")
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--streams", type=int, default=None,
                    help="CUDA streams for the step's launches (default 2; 8 for n <= 64)")
    ap.add_argument("--no-group", action="store_true",
                    help="issue the cases as separate calls instead of one grouped call")
    ap.add_argument("--sustained-probe", action="store_true",
                    help="also measure the power-capped (sustained) TF32 peak (~3 s)")
    ap.add_argument("--config", choices=("sweep", "small", "order4", "hooi", "conventional"),
                    default="sweep")
    ap.add_argument("--batch", type=int, default=1000000)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.config != "sweep":
        run_config(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
