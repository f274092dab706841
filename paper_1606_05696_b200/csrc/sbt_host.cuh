// Host-buffer seam (the reference's numpy-buffer cores, _loops_numba.py:12-68,
// called from kernels.py:107,174,223): copy the touched spans to HBM, one
// launch, copy C back, synchronise.
//
// Re-entrant: every (host thread, device) pair owns a HostCtx -- its own
// non-blocking stream, a grow-only device arena and pinned staging slots -- so
// the reference's `threads > 1` batch chunks (kernels.py:245-266), issued
// concurrently from a ThreadPoolExecutor, overlap one call's copies with
// another's kernel on the GPU instead of serialising on one mutex.
//
// Copies: a span in page-locked memory (cudaHostAlloc / registered, e.g. a
// numpy view of a pinned torch buffer) is DMA'd directly.  A pageable span is
// streamed through 3 pinned slots: the host copies chunk i into a slot (split
// over a small worker pool) while the copy engine moves chunk i-1, so the PCIe
// transfer and the host memcpy overlap.
#pragma once
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "sbt_common.cuh"

namespace sbt {
namespace host {

// ---- a small pool for parallel host memcpy ---------------------------------
class CopyPool {
 public:
  static CopyPool& get() {
    // never destroyed: the detached workers wait on cv_ for the life of the
    // process, and destroying a condition variable with waiters at exit
    // blocks (glibc) -- the process would hang in its static destructors
    static CopyPool* pool = new CopyPool;
    return *pool;
  }
  // memcpy split into `parts` pieces run on the workers (and this thread)
  void copy(void* dst, const void* src, size_t bytes) {
    const size_t min_piece = size_t(1) << 20;
    int parts = int(bytes / min_piece);
    if (parts > nworkers_ + 1) parts = nworkers_ + 1;
    if (parts <= 1) {
      std::memcpy(dst, src, bytes);
      return;
    }
    const size_t piece = ((bytes + parts - 1) / parts + 63) & ~size_t(63);
    std::mutex mu;
    std::condition_variable cv;
    int left = parts - 1;
    for (int i = 1; i < parts; ++i) {
      const size_t off = piece * i;
      const size_t len = off >= bytes ? 0 : (bytes - off < piece ? bytes - off : piece);
      submit([=, &mu, &cv, &left] {
        if (len) std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, len);
        std::lock_guard<std::mutex> g(mu);
        if (--left == 0) cv.notify_one();
      });
    }
    std::memcpy(dst, src, piece < bytes ? piece : bytes);
    std::unique_lock<std::mutex> g(mu);
    cv.wait(g, [&] { return left == 0; });
  }

 private:
  CopyPool() {
    unsigned hc = std::thread::hardware_concurrency();
    nworkers_ = hc > 2 ? int(hc / 2) : 1;
    if (nworkers_ > 16) nworkers_ = 16;
    for (int i = 0; i < nworkers_; ++i)
      std::thread([this] { loop(); }).detach();  // process-lifetime workers
  }
  void submit(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> g(mu_);
      q_.push_back(std::move(f));
    }
    cv_.notify_one();
  }
  void loop() {
    for (;;) {
      std::function<void()> f;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [this] { return !q_.empty(); });
        f = std::move(q_.front());
        q_.erase(q_.begin());
      }
      f();
    }
  }
  int nworkers_ = 1;
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<std::function<void()>> q_;
};

// ---- per (thread, device) context --------------------------------------------
constexpr int kSlots = 3;
constexpr size_t kSlotBytes = size_t(16) << 20;

struct HostCtx {
  int device = -1;
  cudaStream_t stream = nullptr;
  void* arena = nullptr;
  size_t arena_bytes = 0;
  void* slot[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  uint32_t next_slot = 0;  // staging slots rotate across calls: a slot is
                           // refilled only after its last copy drained
  bool ok = false;

  explicit HostCtx(int dev) : device(dev) {
    ok = cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking) == cudaSuccess;
    for (int i = 0; ok && i < kSlots; ++i) {
      ok = cudaHostAlloc(&slot[i], kSlotBytes, cudaHostAllocDefault) == cudaSuccess &&
           cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) == cudaSuccess;
    }
  }
  // device memory for this call (grow-only; the previous arena is freed after
  // this context's stream drained -- every call synchronises before returning)
  cudaError_t reserve(size_t bytes) {
    if (bytes <= arena_bytes) return cudaSuccess;
    if (arena) cudaFree(arena);
    arena = nullptr;
    arena_bytes = 0;
    const size_t want = bytes + bytes / 8;
    cudaError_t e = cudaMalloc(&arena, want);
    if (e == cudaSuccess) arena_bytes = want;
    return e;
  }
};

inline HostCtx* ctx_for_current_device(cudaError_t* err) {
  constexpr int kMaxDev = 64;
  thread_local HostCtx* per_dev[kMaxDev] = {};
  int dev = 0;
  *err = cudaGetDevice(&dev);
  if (*err != cudaSuccess) return nullptr;
  if (dev < 0 || dev >= kMaxDev) {
    *err = cudaErrorInvalidDevice;
    return nullptr;
  }
  if (!per_dev[dev]) per_dev[dev] = new HostCtx(dev);  // lives as long as the thread
  if (!per_dev[dev]->ok) {
    *err = cudaGetLastError();
    if (*err == cudaSuccess) *err = cudaErrorMemoryAllocation;
    return nullptr;
  }
  return per_dev[dev];
}

inline bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// host -> device (span of `bytes` at src)
inline cudaError_t upload(HostCtx* cx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  if (is_pinned(src)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, cx->stream);
  cudaError_t e = cudaSuccess;
  for (size_t off = 0; off < bytes; off += kSlotBytes) {
    // the slot's previous H2D copy (this call or an earlier upload of the same
    // call sequence, e.g. A before B) must have read it before the host
    // overwrites it; an event never recorded completes immediately
    const int s = int(cx->next_slot++ % kSlots);
    const size_t len = bytes - off < kSlotBytes ? bytes - off : kSlotBytes;
    if ((e = cudaEventSynchronize(cx->ev[s])) != cudaSuccess) return e;
    CopyPool::get().copy(cx->slot[s], static_cast<const char*>(src) + off, len);
    if ((e = cudaMemcpyAsync(static_cast<char*>(dst) + off, cx->slot[s], len,
                             cudaMemcpyHostToDevice, cx->stream)) != cudaSuccess)
      return e;
    if ((e = cudaEventRecord(cx->ev[s], cx->stream)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// device -> host, after the work queued on cx->stream; returns after the data
// is in dst
inline cudaError_t download(HostCtx* cx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaStreamSynchronize(cx->stream);
  cudaError_t e;
  if (is_pinned(dst)) {
    if ((e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, cx->stream)) != cudaSuccess)
      return e;
    return cudaStreamSynchronize(cx->stream);
  }
  const size_t nch = (bytes + kSlotBytes - 1) / kSlotBytes;
  auto issue = [&](size_t c) -> cudaError_t {
    const int s = int(c % kSlots);
    const size_t off = c * kSlotBytes;
    const size_t len = bytes - off < kSlotBytes ? bytes - off : kSlotBytes;
    cudaError_t r = cudaMemcpyAsync(cx->slot[s], static_cast<const char*>(src) + off, len,
                                    cudaMemcpyDeviceToHost, cx->stream);
    if (r != cudaSuccess) return r;
    return cudaEventRecord(cx->ev[s], cx->stream);
  };
  // keep kSlots - 1 chunks in flight ahead of the host copy-out
  size_t issued = 0;
  for (; issued < nch && issued < size_t(kSlots - 1); ++issued)
    if ((e = issue(issued)) != cudaSuccess) return e;
  for (size_t c = 0; c < nch; ++c) {
    if (issued < nch) {
      if ((e = issue(issued)) != cudaSuccess) return e;
      ++issued;
    }
    const int s = int(c % kSlots);
    if ((e = cudaEventSynchronize(cx->ev[s])) != cudaSuccess) return e;
    const size_t off = c * kSlotBytes;
    const size_t len = bytes - off < kSlotBytes ? bytes - off : kSlotBytes;
    CopyPool::get().copy(static_cast<char*>(dst) + off, cx->slot[s], len);
  }
  return cudaStreamSynchronize(cx->stream);
}

}  // namespace host
}  // namespace sbt
