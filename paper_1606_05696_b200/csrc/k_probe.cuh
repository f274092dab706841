// Peak-throughput probes for the fp64 roofline denominator (MEASURED_PEAKS.json
// has only copy bandwidth and bf16 GEMM): a register-resident DMMA loop and a
// DFMA loop, each with enough independent chains to saturate the pipe.
#pragma once
#include "sbt_common.cuh"
#include "sm100_ptx.cuh"

namespace sbt {
namespace probe {

__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
  double acc[8][2];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;  // keep the loop alive
}

__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters) {
  double acc[8];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}

// tcgen05 TF32 tensor-pipe peak (the fp32 roofline denominator: 3xTF32 runs
// three of these MMAs per output product).  One CTA per SM; one thread issues
// back-to-back tcgen05.mma.cta_group::1.kind::tf32 M=128 N=256 K=8 from a
// zeroed K-major SW128 tile pair (A 128x32, B 256x32 fp32) into one TMEM
// accumulator, then waits for the last one to retire.  Operands are
// pseudo-random (a zero tile draws less power and would overstate the
// sustained clock).
constexpr int kTf32ProbeSmem = (128 + 256) * 128 + 1024 + 64;
__global__ void __launch_bounds__(128, 1) tf32_umma_peak_kernel(int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (128 + 256) * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  // pseudo-random operands in [-1, 1): zeros would under-state the power
  // draw (and so the clock) of a real contraction
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t(i) + 0x9E3779B9u * (blockIdx.x + 1)) * 2654435761u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    reinterpret_cast<float*>(smem)[i] = float(int32_t(h)) * (1.0f / 2147483648.0f);
  }
  ptx::fence_proxy_async_smem();
  if (threadIdx.x < 32) ptx::tmem_alloc(slot, 256);
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar, 1);
    ptx::fence_mbarrier_init();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = ptx::idesc_tf32(128, 256, false, false);
    const uint32_t a = ptx::smem_addr(smem), b = a + 128 * 128;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        ptx::mma_tf32_ss(tmem, ptx::umma_desc(a + 32 * j, 16, 1024, ptx::kLayoutSW128),
                         ptx::umma_desc(b + 32 * j, 16, 1024, ptx::kLayoutSW128), idesc,
                         (it | j) ? 1u : 0u);
    }
    ptx::tc_commit(bar);
    ptx::mbar_wait(bar, 0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tmem, 256);
}

}  // namespace probe
}  // namespace sbt
