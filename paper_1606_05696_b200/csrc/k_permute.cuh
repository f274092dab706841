// Explicit mode permutation (the "conventional" strategy's transposition,
// reference layout.py:202-215 permute_copy): dst is a packed column-major
// tensor whose mode i is src mode perm[i].
//
// This is NOT on the single-mode hot path -- the planned path never moves an
// operand.  It exists so the paper's comparison (transpose + GEMM versus
// strided batched GEMM, Fig. 1/4; reference planner.py:411-465,
// 620-713) can be run on the device.  It is written to run at HBM speed so the
// comparison is fair to the conventional approach:
//   * if dst mode 0 is also src's unit-stride mode, every warp copies a
//     contiguous run (coalesced both ways);
//   * otherwise a 32 x 32 tile of (dst mode 0, dst mode j) -- j the mode that is
//     unit-stride in src -- goes through shared memory, so reads are coalesced
//     along src's contiguous mode and writes along dst's.
// All remaining modes index the grid (flattened, 64-bit).
#pragma once
#include "sbt_common.cuh"

namespace sbt {
namespace perm {

constexpr int kMaxOrder = 8;

struct PermParams {
  int order;
  int inner;                  // dst mode whose src stride is 1 (0: dst mode 0 itself, or none)
  int64_t dims[kMaxOrder];    // dst extents
  int64_t sstr[kMaxOrder];    // src element stride of each dst mode
  int64_t dstr[kMaxOrder];    // dst (packed) element strides
  int64_t outer;              // product of the extents of the grid modes
};

// decompose the flattened outer index over every mode except 0 and `inner`
__device__ __forceinline__ void outer_offsets(const PermParams& q, int64_t o, int64_t& so,
                                              int64_t& dO) {
  so = 0;
  dO = 0;
  for (int i = 1; i < q.order; ++i) {
    if (i == q.inner) continue;
    const int64_t idx = o % q.dims[i];
    o /= q.dims[i];
    so += idx * q.sstr[i];
    dO += idx * q.dstr[i];
  }
}

// dst mode 0 is src-contiguous (or no mode is): rows of dims[0] copied with
// 256 threads striding the row
template <typename T>
__global__ void __launch_bounds__(256) permute_rows_kernel(const T* __restrict__ src,
                                                           T* __restrict__ dst, PermParams q) {
  const int64_t rows = q.outer;
  const int64_t n0 = q.dims[0];
  for (int64_t o = blockIdx.x; o < rows; o += gridDim.x) {
    int64_t so, dO;
    outer_offsets(q, o, so, dO);
    for (int64_t i = threadIdx.x; i < n0; i += blockDim.x)
      dst[dO + i] = src[so + i * q.sstr[0]];
  }
}

// 32 x 32 tiles over (dst mode 0 = x, dst mode `inner` = y)
template <typename T>
__global__ void __launch_bounds__(256) permute_tile_kernel(const T* __restrict__ src,
                                                           T* __restrict__ dst, PermParams q) {
  __shared__ T tile[32][33];
  const int64_t nx = q.dims[0], ny = q.dims[q.inner];
  const int64_t tx = (nx + 31) / 32, ty = (ny + 31) / 32;
  const int64_t ntiles = tx * ty * q.outer;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;  // 32 x 8 threads
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t bx = t % tx, by = (t / tx) % ty, o = t / (tx * ty);
    int64_t so, dO;
    outer_offsets(q, o, so, dO);
    const int64_t x0 = bx * 32, y0 = by * 32;
    // read: threads along y (src unit stride), rows of x
#pragma unroll
    for (int r = 0; r < 32; r += 8) {
      const int64_t x = x0 + ly + r, y = y0 + lx;
      if (x < nx && y < ny) tile[ly + r][lx] = src[so + x * q.sstr[0] + y];
    }
    __syncthreads();
    // write: threads along x (dst unit stride)
#pragma unroll
    for (int r = 0; r < 32; r += 8) {
      const int64_t y = y0 + ly + r, x = x0 + lx;
      if (x < nx && y < ny) dst[dO + x + y * q.dstr[q.inner]] = tile[lx][ly + r];
    }
    __syncthreads();
  }
}

}  // namespace perm
}  // namespace sbt
