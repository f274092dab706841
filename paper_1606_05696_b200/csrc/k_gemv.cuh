// GEMV-shaped strided batched products (n == 1): y = alpha * A x + beta * y
// per batch entry -- the reference's level-2 kernels (kernels.py:111-153,
// gemv) as used by the batched-GEMV comparison strategy (planner.py:374-404,
// 584-617), and any GEMM call whose N extent is 1.
//
// HBM-bound (one pass over A), so the kernels only have to stream A
// coalesced:
//   * rows contiguous (ars == 1): one thread per row, the warp walks k --
//     every load instruction reads 32 consecutive rows of one column;
//   * k contiguous (acs == 1): one warp per row, lanes stride k, shuffle
//     reduction;
// Accumulation is fp64 for both dtypes (free in a bandwidth-bound kernel;
// keeps fp32 results within the 1e-5 tolerance for any K).
#pragma once
#include "sbt_common.cuh"

namespace sbt {
namespace gemv {

constexpr int kThreads = 256;

template <typename T>
__device__ __forceinline__ void finish(T* y, double acc, T alpha, T beta) {
  const T v = T(acc);
  if (beta == T(0)) *y = alpha * v;
  else *y = alpha * v + beta * *y;
}

// thread per row; grid-stride over (row block, batch, batch2)
template <typename T>
__global__ void __launch_bounds__(kThreads) gemv_rows_kernel(GemmParams<T> p, int64_t nblk) {
  const int64_t total = nblk * p.batch * p.batch2;
  for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
    const int64_t blk = t % nblk, pb = (t / nblk) % p.batch, qb = t / (nblk * p.batch);
    const int64_t i = blk * kThreads + threadIdx.x;
    if (i >= p.m) continue;
    const T* a = p.a + pb * p.aps + qb * p.aps2 + i * p.ars;
    const T* x = p.b + pb * p.bps + qb * p.bps2;
    double acc = 0.0;
    int64_t l = 0;
    for (; l + 4 <= p.k; l += 4) {
      const T a0 = a[l * p.acs], a1 = a[(l + 1) * p.acs], a2 = a[(l + 2) * p.acs],
              a3 = a[(l + 3) * p.acs];
      const T x0 = x[l * p.brs], x1 = x[(l + 1) * p.brs], x2 = x[(l + 2) * p.brs],
              x3 = x[(l + 3) * p.brs];
      acc = fma(double(a0), double(x0), acc);
      acc = fma(double(a1), double(x1), acc);
      acc = fma(double(a2), double(x2), acc);
      acc = fma(double(a3), double(x3), acc);
    }
    for (; l < p.k; ++l) acc = fma(double(a[l * p.acs]), double(x[l * p.brs]), acc);
    finish(p.c + pb * p.cps + qb * p.cps2 + i * p.crs, acc, p.alpha, p.beta);
  }
}

// warp per row, lanes over k (acs == 1)
template <typename T>
__global__ void __launch_bounds__(kThreads) gemv_dot_kernel(GemmParams<T> p) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (kThreads / 32);
  const int64_t total = p.m * p.batch * p.batch2;
  for (int64_t w = int64_t(blockIdx.x) * (kThreads / 32) + (threadIdx.x >> 5); w < total;
       w += warps) {
    const int64_t i = w % p.m, pb = (w / p.m) % p.batch, qb = w / (p.m * p.batch);
    const T* a = p.a + pb * p.aps + qb * p.aps2 + i * p.ars;
    const T* x = p.b + pb * p.bps + qb * p.bps2;
    double acc = 0.0;
    for (int64_t l = lane; l < p.k; l += 32) acc = fma(double(a[l]), double(x[l * p.brs]), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) finish(p.c + pb * p.cps + qb * p.cps2 + i * p.crs, acc, p.alpha, p.beta);
  }
}

}  // namespace gemv
}  // namespace sbt
