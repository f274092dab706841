// C ABI of libsbt200 (declared in include/sbt200.h).
//
// Each extern "C" entry point replaces one function of the reference's
// arithmetic seam (reference backend.py:29-31):
//   sbt_gemm_core_*        <- _loops_numba.py:12-25  gemm_core
//   sbt_batched_core_*     <- _loops_numba.py:28-35  batched_core
//   sbt_ext_batched_core_* <- _loops_numba.py:38-68  ext_batched_core
//   sbt_batched2_core_*    <- planner.py:551-581     LoopStep loop x batched_core
//   sbt_batched_core_host_*  the same over host (numpy) buffers
// The host side validates, picks a kernel family from the stride classes and
// launches exactly one kernel on the caller's stream.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "../../include/sbt200.h"
#include "sbt_common.cuh"
#include "k_generic.cuh"
#include "sbt_dispatch.cuh"
#include "sbt_host.cuh"
#include "k_probe.cuh"
#include "k_permute.cuh"
#include "k_ritz.cuh"
#include "k_gram_apply.cuh"

namespace sbt {

static std::atomic<int64_t> g_launches{0};
static std::atomic<int> g_override{0};
static thread_local std::string t_err;
static thread_local const char* t_last_kernel = "";

static int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}

void note_launch(const char* name) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  t_last_kernel = name;
}

int kernel_override() { return g_override.load(std::memory_order_relaxed); }
static thread_local int t_accumulation = 1;
int accumulation_mode() { return t_accumulation; }

int cuda_fail(cudaError_t e, const char* what) {
  return fail(SBT_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int set_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;  // (kernel, device)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({fn, dev})) return SBT_OK;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(max dynamic smem)");
  done.insert({fn, dev});
  return SBT_OK;
}

static int check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    return fail(SBT_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
  return SBT_OK;
}

template <typename T>
static int validate(const GemmParams<T>& p) {
  if (p.m < 1 || p.n < 1 || p.k < 1)
    return fail(SBT_EINVAL, "extents must be positive (m, n, k >= 1)");
  if (p.batch < 0 || p.batch2 < 0) return fail(SBT_EINVAL, "batch counts must be >= 0");
  const int64_t s[] = {p.ars, p.acs, p.aps, p.aps2, p.brs, p.bcs,
                       p.bps, p.bps2, p.crs, p.ccs, p.cps, p.cps2};
  for (int64_t v : s)
    if (v < 0) return fail(SBT_EINVAL, "strides must be non-negative");
  if (!p.a || !p.b || !p.c) return fail(SBT_EINVAL, "null buffer pointer");
  return SBT_OK;
}

template <typename T>
static int run(GemmParams<T> p, cudaStream_t stream) {
  int rc = validate(p);
  if (rc != SBT_OK) return rc;
  if (p.batch == 0 || p.batch2 == 0) return SBT_OK;  // reference: batch 0 is a no-op
  t_err.clear();
  rc = launch_gemm<T>(p, stream);
  if (rc != SBT_OK) {
    if (t_err.empty())
      return fail(rc, rc == SBT_EUNSUPPORTED ? "no kernel for this request (grid too large)"
                                             : "kernel launch failed");
    return rc;
  }
  return check_cuda(cudaGetLastError(), "kernel launch");
}

template <typename T>
static GemmParams<T> make(int64_t m, int64_t n, int64_t k, T alpha, const T* a, int64_t oa,
                          int64_t ars, int64_t acs, int64_t apt, int64_t apt2, const T* b,
                          int64_t ob, int64_t brs, int64_t bcs, int64_t bpt, int64_t bpt2, T beta,
                          T* c, int64_t oc, int64_t crs, int64_t ccs, int64_t cpt, int64_t cpt2,
                          int64_t batch, int64_t batch2) {
  GemmParams<T> p;
  p.m = m; p.n = n; p.k = k; p.batch = batch; p.batch2 = batch2;
  p.a = a ? a + oa : nullptr; p.ars = ars; p.acs = acs; p.aps = apt; p.aps2 = apt2;
  p.b = b ? b + ob : nullptr; p.brs = brs; p.bcs = bcs; p.bps = bpt; p.bps2 = bpt2;
  p.c = c ? c + oc : nullptr; p.crs = crs; p.ccs = ccs; p.cps = cpt; p.cps2 = cpt2;
  p.alpha = alpha; p.beta = beta;
  if (oa < 0 || ob < 0 || oc < 0) { p.m = -1; }  // rejected by validate()
  return p;
}

template <typename T>
static GemmParams<T> from_desc(const sbt_gemm_desc& d) {
  return make<T>(d.m, d.n, d.k, T(d.alpha), static_cast<const T*>(d.a), d.oa, d.ars, d.acs,
                 d.apt, d.apt2, static_cast<const T*>(d.b), d.ob, d.brs, d.bcs, d.bpt, d.bpt2,
                 T(d.beta), static_cast<T*>(d.c), d.oc, d.crs, d.ccs, d.cpt, d.cpt2, d.batch,
                 d.batch2);
}

// Grouped execution: see include/sbt200.h.  fp32 problems the pair kernel
// takes are bucketed by kernel configuration and launched together.
template <bool SPLIT, bool BB, int BNT>
struct GroupRun {
  static int run(const std::vector<PairPlan>& plans, const std::vector<int>& idx,
                 cudaStream_t stream, std::vector<char>& launched) {
    bool* flags = reinterpret_cast<bool*>(launched.data());
    return GroupLaunch<SPLIT, BB, BNT>::run(plans.data(), idx.data(), int(idx.size()), stream,
                                            flags);
  }
};

// internal streams for forking independent launches of a group (per host
// thread; the events are re-recorded on every call)
constexpr int kForkLanes = 8;
struct ForkStreams {
  cudaStream_t s[kForkLanes];
  cudaEvent_t fork, join[kForkLanes];
  bool ok = true;
  ForkStreams() {
    for (int l = 0; l < kForkLanes; ++l) {
      ok = ok && cudaStreamCreateWithFlags(&s[l], cudaStreamNonBlocking) == cudaSuccess;
      ok = ok && cudaEventCreateWithFlags(&join[l], cudaEventDisableTiming) == cudaSuccess;
    }
    ok = ok && cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess;
    if (!ok) cudaGetLastError();  // e.g. first use inside a stream capture: stay serial
  }
};
// one lane set per (host thread, device): streams belong to the device that
// was current when they were created
constexpr int kMaxDevices = 64;
static ForkStreams* fork_streams() {
  thread_local ForkStreams* per_dev[kMaxDevices] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    cudaGetLastError();
    return nullptr;
  }
  if (!per_dev[dev]) per_dev[dev] = new ForkStreams();  // lives as long as the thread
  return per_dev[dev]->ok ? per_dev[dev] : nullptr;
}

template <typename T>
static int run_group(int count, const sbt_gemm_desc* descs, cudaStream_t stream_in) {
  const cudaStream_t stream = stream_in;
  if (count < 0 || (count > 0 && !descs)) return fail(SBT_EINVAL, "group: bad arguments");
  std::vector<GemmParams<T>> ps;
  ps.reserve(count);
  for (int i = 0; i < count; ++i) {
    GemmParams<T> p = from_desc<T>(descs[i]);
    const int rc = validate(p);
    if (rc != SBT_OK) return rc;
    ps.push_back(p);
  }
  std::vector<char> launched(count, 0);
  // fork point before any launch: forked calls (below) then overlap the
  // grouped launches instead of queueing behind them
  ForkStreams* fs = count >= 2 ? fork_streams() : nullptr;
  if (fs && cudaEventRecord(fs->fork, stream) != cudaSuccess) {
    cudaGetLastError();
    fs = nullptr;  // serial issue
  }
  bool forked = false;
  // join the internal lanes back into the caller's stream on EVERY exit path
  // (an unjoined lane would invalidate an enclosing stream capture)
  auto finish = [&](int rc) -> int {
    if (forked) {
      for (int l = 0; l < kForkLanes; ++l) {
        const cudaError_t e1 = cudaEventRecord(fs->join[l], fs->s[l]);
        const cudaError_t e2 = cudaStreamWaitEvent(stream, fs->join[l], 0);
        if (rc == SBT_OK && e1 != cudaSuccess) rc = cuda_fail(e1, "group join (event record)");
        if (rc == SBT_OK && e2 != cudaSuccess) rc = cuda_fail(e2, "group join (stream wait)");
      }
      forked = false;
    }
    if (rc != SBT_OK) return rc;
    return check_cuda(cudaGetLastError(), "group launch");
  };
  int lane_next = 0;
  auto lane = [&]() -> cudaStream_t {  // next internal stream (joined at the end)
    if (!forked) {
      for (int l = 0; l < kForkLanes; ++l) cudaStreamWaitEvent(fs->s[l], fs->fork, 0);
      forked = true;  // (a failed wait surfaces in the final cudaGetLastError check)
    }
    return fs->s[(lane_next++) % kForkLanes];
  };
  if constexpr (sizeof(T) == 4) {
    if (kernel_override() == 0) {
      // bucket the pair-kernel problems by configuration (bb, split, bnt)
      std::vector<PairPlan> plans(count);
      std::vector<int> buckets[12];
      for (int i = 0; i < count; ++i) {
        const GemmParams<float>& p = ps[i];
        if (p.batch == 0 || p.batch2 == 0) { launched[i] = 1; continue; }
        if (p.k > kMaxChunkK) continue;                       // K-chunked: single path
        if (!plan_pair(p, &plans[i])) continue;
        const PairPlan& pl = plans[i];
        const int key = pl.bb ? (8 + (pl.bnt == 128 ? 2 : 0) + (pl.split ? 1 : 0))
                              : ((pl.bnt == 32 ? 0 : pl.bnt == 64 ? 1 : pl.bnt == 128 ? 2 : 3) * 2 +
                                 (pl.split ? 1 : 0));
        buckets[key].push_back(i);
      }
      int nbuckets = 0;
      for (int key = 0; key < 12; ++key) nbuckets += buckets[key].empty() ? 0 : 1;
      for (int key = 0; key < 12; ++key) {
        if (buckets[key].empty()) continue;
        const PairPlan& pl0 = plans[buckets[key][0]];
        // independent configurations: their persistent launches overlap
        // each other's tails on separate internal streams
        const cudaStream_t stream = (fs && nbuckets >= 2) ? lane() : stream_in;
        int rc;
        if (pl0.bb && pl0.bnt == 128) {
          rc = pl0.split ? GroupRun<true, true, 128>::run(plans, buckets[key], stream, launched)
                         : GroupRun<false, true, 128>::run(plans, buckets[key], stream, launched);
        } else if (pl0.bb) {
          rc = pl0.split ? GroupRun<true, true, 256>::run(plans, buckets[key], stream, launched)
                         : GroupRun<false, true, 256>::run(plans, buckets[key], stream, launched);
        } else {
          switch (pl0.bnt) {
            case 32: rc = pl0.split ? GroupRun<true, false, 32>::run(plans, buckets[key], stream, launched)
                                    : GroupRun<false, false, 32>::run(plans, buckets[key], stream, launched); break;
            case 64: rc = pl0.split ? GroupRun<true, false, 64>::run(plans, buckets[key], stream, launched)
                                    : GroupRun<false, false, 64>::run(plans, buckets[key], stream, launched); break;
            case 128: rc = pl0.split ? GroupRun<true, false, 128>::run(plans, buckets[key], stream, launched)
                                     : GroupRun<false, false, 128>::run(plans, buckets[key], stream, launched); break;
            default: rc = pl0.split ? GroupRun<true, false, 256>::run(plans, buckets[key], stream, launched)
                                    : GroupRun<false, false, 256>::run(plans, buckets[key], stream, launched); break;
          }
        }
        if (rc < 0) return finish(rc);
      }
    }
  }
  // everything not grouped: one call each.  Many of them (small problems whose
  // launches are mostly latency) fork onto internal streams and join back, so
  // independent launches overlap on the GPU (capturable: event fork / join)
  std::vector<int> rest;
  for (int i = 0; i < count; ++i)
    if (!launched[i]) rest.push_back(i);
  const bool fork_rest = fs && (rest.size() >= 2 || (forked && !rest.empty()));
  for (int i : rest) {
    const int rc = run<T>(ps[i], fork_rest ? lane() : stream);
    if (rc != SBT_OK) return finish(rc);
  }
  return finish(SBT_OK);
}

// ---- host-buffer path (re-entrant: see sbt_host.cuh) -------------------------
static int64_t span_of(int64_t m, int64_t k, int64_t rs, int64_t cs, int64_t ps, int64_t batch) {
  return 1 + (m - 1) * rs + (k - 1) * cs + (batch > 0 ? (batch - 1) * ps : 0);
}

template <typename T>
static int run_host(int64_t m, int64_t n, int64_t k, T alpha, const T* a, int64_t oa,
                    int64_t ars, int64_t acs, int64_t apt, const T* b, int64_t ob, int64_t brs,
                    int64_t bcs, int64_t bpt, T beta, T* c, int64_t oc, int64_t crs, int64_t ccs,
                    int64_t cpt, int64_t batch) {
  GemmParams<T> probe = make<T>(m, n, k, alpha, a, oa, ars, acs, apt, 0, b, ob, brs, bcs, bpt,
                                0, beta, c, oc, crs, ccs, cpt, 0, batch, 1);
  int rc = validate(probe);
  if (rc != SBT_OK) return rc;
  if (batch == 0) return SBT_OK;
  const int64_t na = span_of(m, k, ars, acs, apt, batch);
  const int64_t nb = span_of(k, n, brs, bcs, bpt, batch);
  const int64_t nc = span_of(m, n, crs, ccs, cpt, batch);
  const bool c_dense = (nc == m * n * batch);
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t ba = align(na * sizeof(T)), bb = align(nb * sizeof(T)), bc = align(nc * sizeof(T));
  cudaError_t e = cudaSuccess;
  host::HostCtx* cx = host::ctx_for_current_device(&e);
  if (!cx) return cuda_fail(e, "host seam: per-thread stream / staging buffers");
  if ((e = cx->reserve(ba + bb + bc)) != cudaSuccess) return cuda_fail(e, "host seam: device arena");
  char* base = static_cast<char*>(cx->arena);
  T* da = reinterpret_cast<T*>(base);
  T* db = reinterpret_cast<T*>(base + ba);
  T* dc = reinterpret_cast<T*>(base + ba + bb);
  if ((e = host::upload(cx, da, a + oa, na * sizeof(T))) != cudaSuccess) return cuda_fail(e, "H2D A");
  if ((e = host::upload(cx, db, b + ob, nb * sizeof(T))) != cudaSuccess) return cuda_fail(e, "H2D B");
  // C's span is copied in unless beta == 0 and the batch regions tile it exactly
  // (otherwise the gaps between regions must survive the copy back).
  if (beta != T(0) || !c_dense) {
    if ((e = host::upload(cx, dc, c + oc, nc * sizeof(T))) != cudaSuccess)
      return cuda_fail(e, "H2D C");
  }
  GemmParams<T> p = make<T>(m, n, k, alpha, da, 0, ars, acs, apt, 0, db, 0, brs, bcs, bpt, 0,
                            beta, dc, 0, crs, ccs, cpt, 0, batch, 1);
  if ((rc = run(p, cx->stream)) != SBT_OK) {
    cudaStreamSynchronize(cx->stream);  // leave the context idle for the next call
    return rc;
  }
  if ((e = host::download(cx, c + oc, dc, nc * sizeof(T))) != cudaSuccess)
    return cuda_fail(e, "D2H C");
  return SBT_OK;
}

}  // namespace sbt

using namespace sbt;

namespace sbt {
// Explicit permutation copy (conventional strategy only; see k_permute.cuh).
template <typename T>
static int run_permute(int order, const int64_t* dims, const T* src, const int64_t* sstr, T* dst,
                       cudaStream_t stream) {
  if (order < 1 || order > perm::kMaxOrder || !dims || !sstr || !src || !dst)
    return fail(SBT_EINVAL, "permute: bad arguments");
  perm::PermParams q{};
  q.order = order;
  q.inner = 0;
  int64_t total = 1, d = 1;
  for (int i = 0; i < order; ++i) {
    if (dims[i] < 1 || sstr[i] < 0) return fail(SBT_EINVAL, "permute: bad extent or stride");
    q.dims[i] = dims[i];
    q.sstr[i] = sstr[i];
    q.dstr[i] = d;
    d *= dims[i];
    total *= dims[i];
  }
  if (sstr[0] != 1)
    for (int i = 1; i < order; ++i)
      if (sstr[i] == 1 && dims[i] > 1) { q.inner = i; break; }
  q.outer = total / q.dims[0] / (q.inner ? q.dims[q.inner] : 1);
  int64_t work = q.inner ? ceil_div(q.dims[0], 32) * ceil_div(q.dims[q.inner], 32) * q.outer : q.outer;
  const int64_t grid = work < int64_t(kNumSMs) * 16 ? work : int64_t(kNumSMs) * 16;
  if (q.inner) {
    perm::permute_tile_kernel<T><<<unsigned(grid), 256, 0, stream>>>(src, dst, q);
    note_launch("permute_tile");
  } else {
    perm::permute_rows_kernel<T><<<unsigned(grid), 256, 0, stream>>>(src, dst, q);
    note_launch("permute_rows");
  }
  return check_cuda(cudaGetLastError(), "permute launch");
}

}  // namespace sbt

extern "C" {

int sbt_version(void) { return 100; }
const char* sbt_last_error(void) { return t_err.c_str(); }
int64_t sbt_launch_count(void) { return g_launches.load(); }
const char* sbt_last_kernel(void) { return t_last_kernel; }
int sbt_set_kernel_override(int which) {
  if (which < 0 || which > 3) return SBT_EINVAL;
  g_override.store(which);
  return SBT_OK;
}
int sbt_set_accumulation(int mode) {
  const int prev = t_accumulation;
  t_accumulation = mode ? 1 : 0;
  return prev;
}

// Diagnostics: measured fp64 tensor (kind 0 = DMMA) or SIMT (kind 1 = DFMA)
// throughput in TFLOP/s on the current device.  Not part of the reference seam.
int sbt_probe_fp64_peak(int kind, double* tflops) {
  if (!tflops || kind < 0 || kind > 1) return fail(SBT_EINVAL, "bad probe arguments");
  double* out = nullptr;
  int rc;
  if ((rc = check_cuda(cudaMalloc(&out, sizeof(double)), "cudaMalloc")) != SBT_OK) return rc;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, blocks = kNumSMs * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {  // first launch warms up
    cudaEventRecord(e0);
    if (kind == 0) probe::dmma_peak_kernel<<<blocks, threads>>>(out, iters);
    else probe::dfma_peak_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
  }
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = double(blocks) * threads / 32.0;
  // DMMA m8n8k4: 256 FMA per warp instruction; DFMA: 32 FMA per warp instruction
  const double fma = warps * iters * 8.0 * (kind == 0 ? 256.0 : 32.0);
  *tflops = 2.0 * fma / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  note_launch(kind == 0 ? "probe_dmma" : "probe_dfma");
  return check_cuda(cudaGetLastError(), "probe");
}

// Diagnostics: measured dense TF32 tensor-pipe throughput (tcgen05.mma
// kind::tf32) in TFLOP/s on the current device; 3xTF32 peak = this / 3.
int sbt_probe_tf32_peak(double* tflops) {
  if (!tflops) return fail(SBT_EINVAL, "bad probe arguments");
  auto kern = probe::tf32_umma_peak_kernel;
  int rc;
  if ((rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            probe::kTf32ProbeSmem),
                       "cudaFuncSetAttribute")) != SBT_OK)
    return rc;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 8192, blocks = kNumSMs;
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {  // first launch warms up; keep the fastest
    cudaEventRecord(e0);
    kern<<<blocks, 128, probe::kTf32ProbeSmem>>>(iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  // 4 MMAs of M=128 N=256 K=8 per iteration per CTA
  const double flops = 2.0 * blocks * double(iters) * 4.0 * 128 * 256 * 8;
  *tflops = flops / (best * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  note_launch("probe_tf32_umma");
  return check_cuda(cudaGetLastError(), "probe");
}

// Sustained variant: back-to-back probe launches for `seconds` (clocks settle
// under the power cap), throughput of the second half.
int sbt_probe_tf32_sustained(double seconds, double* tflops) {
  if (!tflops || !(seconds > 0.0) || seconds > 60.0)
    return fail(SBT_EINVAL, "bad probe arguments");
  auto kern = probe::tf32_umma_peak_kernel;
  int rc;
  if ((rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            probe::kTf32ProbeSmem),
                       "cudaFuncSetAttribute")) != SBT_OK)
    return rc;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 8192, blocks = kNumSMs;
  const double flops_per_launch = 2.0 * blocks * double(iters) * 4.0 * 128 * 256 * 8;
  // one launch is ~3 ms at full clock: size the two halves from that
  const int half = int(seconds / 2 / 3e-3) + 1;
  for (int i = 0; i < half; ++i) kern<<<blocks, 128, probe::kTf32ProbeSmem>>>(iters);
  cudaEventRecord(e0);
  for (int i = 0; i < half; ++i) kern<<<blocks, 128, probe::kTf32ProbeSmem>>>(iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *tflops = flops_per_launch * half / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  note_launch("probe_tf32_umma");
  return check_cuda(cudaGetLastError(), "probe");
}

int sbt_batched_core_group_f32(int count, const sbt_gemm_desc* descs, void* stream) {
  return sbt::run_group<float>(count, descs, (cudaStream_t)stream);
}
int sbt_batched_core_group_f64(int count, const sbt_gemm_desc* descs, void* stream) {
  return sbt::run_group<double>(count, descs, (cudaStream_t)stream);
}

int sbt_permute_f64(int order, const int64_t* dims, const double* src, const int64_t* src_strides,
                    double* dst, void* stream) {
  return sbt::run_permute<double>(order, dims, src, src_strides, dst, (cudaStream_t)stream);
}
int sbt_permute_f32(int order, const int64_t* dims, const float* src, const int64_t* src_strides,
                    float* dst, void* stream) {
  return sbt::run_permute<float>(order, dims, src, src_strides, dst, (cudaStream_t)stream);
}

#define SBT_DEFINE(T, SUF)                                                                     \
  int sbt_gemm_core_##SUF(int64_t m, int64_t n, int64_t k, T alpha, const T* a, int64_t oa,     \
                          int64_t ars, int64_t acs, const T* b, int64_t ob, int64_t brs,        \
                          int64_t bcs, T beta, T* c, int64_t oc, int64_t crs, int64_t ccs,      \
                          void* stream) {                                                       \
    return run(make<T>(m, n, k, alpha, a, oa, ars, acs, 0, 0, b, ob, brs, bcs, 0, 0, beta, c,   \
                       oc, crs, ccs, 0, 0, 1, 1),                                               \
               (cudaStream_t)stream);                                                           \
  }                                                                                             \
  int sbt_batched_core_##SUF(int64_t m, int64_t n, int64_t k, T alpha, const T* a, int64_t oa,  \
                             int64_t ars, int64_t acs, int64_t apt, const T* b, int64_t ob,     \
                             int64_t brs, int64_t bcs, int64_t bpt, T beta, T* c, int64_t oc,   \
                             int64_t crs, int64_t ccs, int64_t cpt, int64_t batch,              \
                             void* stream) {                                                    \
    return run(make<T>(m, n, k, alpha, a, oa, ars, acs, apt, 0, b, ob, brs, bcs, bpt, 0, beta,  \
                       c, oc, crs, ccs, cpt, 0, batch, 1),                                      \
               (cudaStream_t)stream);                                                           \
  }                                                                                             \
  int sbt_ext_batched_core_##SUF(int64_t m, int64_t n, int64_t k, T alpha, const T* a,          \
                                 int64_t oa, int64_t ars, int64_t acs, int64_t apt, const T* b, \
                                 int64_t ob, int64_t brs, int64_t bcs, int64_t bpt, T beta,     \
                                 T* c, int64_t oc, int64_t crs, int64_t ccs, int64_t cpt,       \
                                 int64_t batch, void* stream) {                                 \
    return run(make<T>(m, n, k, alpha, a, oa, ars, acs, apt, 0, b, ob, brs, bcs, bpt, 0, beta,  \
                       c, oc, crs, ccs, cpt, 0, batch, 1),                                      \
               (cudaStream_t)stream);                                                           \
  }                                                                                             \
  int sbt_batched2_core_##SUF(int64_t m, int64_t n, int64_t k, T alpha, const T* a, int64_t oa, \
                              int64_t ars, int64_t acs, int64_t apt, int64_t apt2, const T* b,  \
                              int64_t ob, int64_t brs, int64_t bcs, int64_t bpt, int64_t bpt2,  \
                              T beta, T* c, int64_t oc, int64_t crs, int64_t ccs, int64_t cpt,  \
                              int64_t cpt2, int64_t batch, int64_t batch2, void* stream) {      \
    return run(make<T>(m, n, k, alpha, a, oa, ars, acs, apt, apt2, b, ob, brs, bcs, bpt, bpt2,  \
                       beta, c, oc, crs, ccs, cpt, cpt2, batch, batch2),                        \
               (cudaStream_t)stream);                                                           \
  }                                                                                             \
  int sbt_batched_core_host_##SUF(int64_t m, int64_t n, int64_t k, T alpha, const T* a,         \
                                  int64_t oa, int64_t ars, int64_t acs, int64_t apt,            \
                                  const T* b, int64_t ob, int64_t brs, int64_t bcs,             \
                                  int64_t bpt, T beta, T* c, int64_t oc, int64_t crs,           \
                                  int64_t ccs, int64_t cpt, int64_t batch) {                    \
    return run_host<T>(m, n, k, alpha, a, oa, ars, acs, apt, b, ob, brs, bcs, bpt, beta, c, oc, \
                       crs, ccs, cpt, batch);                                                   \
  }

SBT_DEFINE(double, f64)
SBT_DEFINE(float, f32)

// Rayleigh-Ritz finish of one warm-started subspace sweep (HOOI factor
// update, reference tucker.py:63-76); see k_ritz.cuh.  Asynchronous: the
// convergence flag is read by the caller later.
int sbt_ritz_f64(const double* qz, const double* m, int64_t n, int p, int rank, double tol,
                 double* ut, double* yt, float* ut32, double* w, int* flag, double* rel,
                 void* stream) {
  if (!qz || !ut || !w || !flag || !rel || n < 1 || p < 1 || p > ritz::kMaxP ||
      rank < 1 || rank > p || p > n)
    return fail(SBT_EINVAL, "sbt_ritz_f64: bad arguments");
  {
    const int rc = set_smem_attr(reinterpret_cast<const void*>(ritz::ritz_kernel), ritz::SMEM_BYTES);
    if (rc != SBT_OK) return rc;
  }
  ritz::ritz_kernel<<<ritz::kCluster, ritz::kThreads, ritz::SMEM_BYTES, static_cast<cudaStream_t>(stream)>>>(
      qz, n, qz + int64_t(p) * n, n, m, n, p, rank, tol, ut, yt, ut32, w, flag, rel);
  note_launch("ritz");
  return check_cuda(cudaGetLastError(), "ritz launch");
}

}  // extern "C"

namespace {

// the unfolding geometry of a packed tensor (k_gram_apply.cuh)
int unfold_of(int order, const int64_t* dims, int mode, sbt::gapply::Unfold& u) {
  if (order < 1 || order > 16 || !dims || mode < 0 || mode >= order) return -1;
  int64_t a = 1, total = 1;  // (the kernels keep A = prod(d_<mode) in 32 bits)
  for (int i = 0; i < order; ++i) {
    if (dims[i] < 1) return -1;
    if (i < mode) a *= dims[i];
    total *= dims[i];
  }
  u.n = dims[mode];
  u.cols = total / u.n;
  u.A = a;
  return a < (int64_t(1) << 31) ? 0 : -1;
}

template <typename TY, typename TO, bool MODE_OUT>
int launch_w(const TY* y, const sbt::gapply::Unfold& u, const double* qt, int64_t ldq, int p,
             TO* out, cudaStream_t stream) {
  using namespace sbt;
  const int ys = int(sizeof(TY));
  const int rch = gapply::w_rows_per_chunk(u.n, p, ys);
  const int smem = int(gapply::w_smem_bytes(rch, p, ys));
  auto kern = gapply::w_kernel<TY, TO, MODE_OUT>;
  // the attribute is set once per (kernel, device): the largest chunk any call uses
  int rc = set_smem_attr(reinterpret_cast<const void*>(kern), gapply::W_SMEM_MAX + 1024);
  if (rc != SBT_OK) return rc;
  // 1-D bulk copies need 16-byte aligned rows of a multiple of 16 bytes
  const bool qbulk = reinterpret_cast<uintptr_t>(qt) % 16 == 0 && ldq % 2 == 0 && u.n % 2 == 0;
  const bool ybulk = u.A == 1 && reinterpret_cast<uintptr_t>(y) % 16 == 0 &&
                     (u.n * ys) % 16 == 0;
  kern<<<unsigned(ceil_div(u.cols, gapply::CB)), gapply::NT, smem, stream>>>(
      y, u, qt, ldq, p, out, rch, (qbulk ? 1 : 0) | (ybulk ? 2 : 0));
  note_launch(MODE_OUT ? "mode_product_acc64" : "gram_apply_w");
  return check_cuda(cudaGetLastError(), "gram_apply w_kernel launch");
}

template <typename TY>
int hooi_factor(const TY* y, int order, const int64_t* dims, int mode, const double* qt,
                int64_t ldq, int p, int rank, double tol, void* ws, size_t ws_bytes, double* ut,
                double* yt, float* ut32, double* w, int* flag, double* rel, void* stream_) {
  using namespace sbt;
  gapply::Unfold u;
  if (!y || !qt || !ws || !ut || !w || !flag || !rel || unfold_of(order, dims, mode, u) ||
      p < 1 || p > gapply::kMaxP || p > ritz::kMaxP || rank < 1 || rank > p || p > u.n ||
      ldq < u.n)
    return fail(SBT_EINVAL, "sbt_hooi_factor: bad arguments");
  const gapply::Plan pl = gapply::plan(u.n, u.cols, p);
  if (ws_bytes < size_t(pl.bytes))
    return fail(SBT_EINVAL, "sbt_hooi_factor: workspace too small (see sbt_hooi_factor_ws_bytes)");
  if (reinterpret_cast<uintptr_t>(ws) % 16)
    return fail(SBT_EINVAL, "sbt_hooi_factor: workspace must be 16-byte aligned");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  double* wsd = static_cast<double*>(ws);
  double* wt = wsd + pl.w_off;
  double* zt = wsd + pl.z_off;
  // diagnostics (tools/factor_bench.py): 1 = W only, 2 = W and Z, else all
  static const int stop_after = env_int("SBT_GA_DEBUG", 0);
  int rc = launch_w<TY, double, false>(y, u, qt, ldq, p, wt, stream);
  if (rc != SBT_OK || stop_after == 1) return rc;
  rc = set_smem_attr(reinterpret_cast<const void*>(gapply::z_kernel<TY>), gapply::Z_SMEM_BYTES);
  if (rc != SBT_OK) return rc;
  gapply::z_kernel<TY><<<dim3(unsigned(pl.tiles), unsigned(gapply::ZS)), gapply::NT,
                         gapply::Z_SMEM_BYTES, stream>>>(y, u, wt, p, pl.kper, zt, u.n);
  note_launch("gram_apply_z");
  rc = check_cuda(cudaGetLastError(), "gram_apply_z launch");
  if (rc != SBT_OK || stop_after == 2) return rc;
  rc = set_smem_attr(reinterpret_cast<const void*>(ritz::ritz_kernel), ritz::SMEM_BYTES);
  if (rc != SBT_OK) return rc;
  ritz::ritz_kernel<<<ritz::kCluster, ritz::kThreads, ritz::SMEM_BYTES, stream>>>(
      qt, ldq, zt, u.n, nullptr, u.n, p, rank, tol, ut, yt, ut32, w, flag, rel);
  note_launch("ritz");
  return check_cuda(cudaGetLastError(), "ritz launch");
}

template <typename T>
int hooi_status(const T* x, int64_t count, const int* flags, int nflags, double* out,
                void* stream) {
  using namespace sbt;
  if (!x || count < 0 || nflags < 0 || nflags > 64 || (nflags && !flags) || !out)
    return fail(SBT_EINVAL, "sbt_hooi_status: bad arguments");
  gapply::status_kernel<T><<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(x, count, flags,
                                                                              nflags, out);
  note_launch("hooi_status");
  return check_cuda(cudaGetLastError(), "hooi_status launch");
}

template <typename T>
int mode_product_acc64(const T* y, int order, const int64_t* dims, int mode, const double* qt,
                       int64_t ldq, int p, T* out, void* stream) {
  using namespace sbt;
  gapply::Unfold u;
  if (!y || !qt || !out || unfold_of(order, dims, mode, u) || p < 1 || p > gapply::kMaxP ||
      ldq < u.n)
    return fail(SBT_EINVAL, "sbt_mode_product_acc64: bad arguments");
  return launch_w<T, T, true>(y, u, qt, ldq, p, out, static_cast<cudaStream_t>(stream));
}

}  // namespace

extern "C" {

#ifdef SBT_TRACE
// diagnostics build only (tools/flush_trace.py): the CTA-pair kernel's timeline
// of the last launch (pair 0): which 0 = g_trace [8][4096], 1 = g_trace_flush
// [2][4096], 2 = g_trace_epi [2][64][4], 3 = g_trace_mma [64][2]
int sbt_trace_dump(int which, long long* out) {
  cudaError_t e = cudaErrorInvalidValue;
  if (which == 0) e = cudaMemcpyFromSymbol(out, sbt::tf32tma::g_trace, sizeof(sbt::tf32tma::g_trace));
  if (which == 1) e = cudaMemcpyFromSymbol(out, sbt::tf32tma::g_trace_flush, sizeof(sbt::tf32tma::g_trace_flush));
  if (which == 2) e = cudaMemcpyFromSymbol(out, sbt::tf32tma::g_trace_epi, sizeof(sbt::tf32tma::g_trace_epi));
  if (which == 3) e = cudaMemcpyFromSymbol(out, sbt::tf32tma::g_trace_mma, sizeof(sbt::tf32tma::g_trace_mma));
  return e == cudaSuccess ? 0 : -3;
}
#endif

#ifdef SBT_RITZ_CLOCK
// diagnostics build only (tools/ritz_probe.py with SBT_LIB): the Ritz
// kernel's phase stamps of the last launch
int sbt_ritz_clock(long long* out) {
  return cudaMemcpyFromSymbol(out, sbt::ritz::g_ritz_clock, 24 * sizeof(long long)) ==
                 cudaSuccess ? 0 : -3;
}
int sbt_ga_clock(long long* out) {
  return (cudaMemcpyFromSymbol(out, sbt::gapply::g_ga_clock, 8 * sizeof(long long)) ==
              cudaSuccess &&
          cudaMemcpyFromSymbol(out + 8, sbt::gapply::g_gz_clock, 8 * sizeof(long long)) ==
              cudaSuccess) ? 0 : -3;
}
#endif

int sbt_mode_product_acc64_f32(const float* y, int order, const int64_t* dims, int mode,
                               const double* qt, int64_t ldq, int p, float* out, void* stream) {
  return mode_product_acc64<float>(y, order, dims, mode, qt, ldq, p, out, stream);
}

int sbt_mode_product_acc64_f64(const double* y, int order, const int64_t* dims, int mode,
                               const double* qt, int64_t ldq, int p, double* out, void* stream) {
  return mode_product_acc64<double>(y, order, dims, mode, qt, ldq, p, out, stream);
}

size_t sbt_hooi_factor_ws_bytes(int order, const int64_t* dims, int mode, int p) {
  sbt::gapply::Unfold u;
  if (unfold_of(order, dims, mode, u) || p < 1 || p > sbt::gapply::kMaxP) return 0;
  return size_t(sbt::gapply::plan(u.n, u.cols, p).bytes);
}

int sbt_hooi_factor_f32(const float* y, int order, const int64_t* dims, int mode,
                        const double* qt, int64_t ldq, int p, int rank, double tol, void* ws,
                        size_t ws_bytes, double* ut, double* yt, float* ut32, double* w,
                        int* flag, double* rel, void* stream) {
  return hooi_factor<float>(y, order, dims, mode, qt, ldq, p, rank, tol, ws, ws_bytes, ut, yt,
                            ut32, w, flag, rel, stream);
}

int sbt_hooi_factor_f64(const double* y, int order, const int64_t* dims, int mode,
                        const double* qt, int64_t ldq, int p, int rank, double tol, void* ws,
                        size_t ws_bytes, double* ut, double* yt, float* ut32, double* w,
                        int* flag, double* rel, void* stream) {
  return hooi_factor<double>(y, order, dims, mode, qt, ldq, p, rank, tol, ws, ws_bytes, ut, yt,
                             ut32, w, flag, rel, stream);
}

int sbt_hooi_status_f32(const float* core, int64_t count, const int* flags, int nflags,
                        double* out, void* stream) {
  return hooi_status<float>(core, count, flags, nflags, out, stream);
}

int sbt_hooi_status_f64(const double* core, int64_t count, const int* flags, int nflags,
                        double* out, void* stream) {
  return hooi_status<double>(core, count, flags, nflags, out, stream);
}

}  // extern "C"
