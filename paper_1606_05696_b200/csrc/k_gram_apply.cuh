// Z = G Q = Y_(r) (Y_(r)^T Q): the Gram-times-basis product of one HOOI
// factor update (reference tucker.py:63-76 takes the leading eigenvectors of
// the mode-r Gram Y_(r) Y_(r)^T; tucker.py:160-167 applies it to the partial
// core Y of each mode), read straight from the packed fp32 / fp64 tensor Y.
//
// For a packed column-major tensor with dims d_0..d_{N-1}, the mode-r
// unfolding needs no copy: with A = prod(d_<r) and n = d_r,
//   Y_(r)[i, c] = y[(c % A) + i * A + (c / A) * A * n]
// (columns ordered mode-0-fastest over the remaining modes; any column order
// gives the same Gram).  fp32 elements are widened to fp64 as they are staged,
// so every product accumulates in fp64 and no fp64 unfolding is materialised.
//
// Two kernels (the second consumes the whole of W):
//   w_kernel : W = Y_(r)^T Q     (cols x p, K = n), one CTA per CB columns;
//   z_kernel : Z = Y_(r) W       (n x p, K = cols), RB-row tiles x S K-splits,
//              partial tiles summed in split order by the last CTA of each
//              tile (atomic ticket, reset by that CTA): deterministic, one
//              launch, no zeroing between graph replays.
// Y is written by the mode product right before, so it is L2-resident; the
// kernels are latency-bound and sized to put ~128 CTAs on the 148 SMs.
#pragma once
#include "sbt_common.cuh"

namespace sbt {
namespace gapply {

constexpr int NT = 256;         // 8 warps
constexpr int kMaxP = 64;       // basis width (lane j and j + 32)
constexpr int CB = 8;           // W columns per CTA
constexpr int TR = 64;          // staged rows (w_kernel) / columns (z_kernel) per step
constexpr int RB = 32;          // Z rows per CTA (4 per warp)
constexpr int TZ = 32;          // staged columns per step (z_kernel)
constexpr int LQ = kMaxP + 1;   // padded row of a staged Q / W tile

struct Unfold {
  int64_t n;     // rows (d_r)
  int64_t cols;  // prod of the other extents
  int64_t A;     // prod(d_<r): unit-stride run of a column index
};

template <typename TY>
__device__ __forceinline__ double yat(const TY* __restrict__ y, const Unfold& u, int64_t i,
                                      int64_t c) {
  const int64_t a = c % u.A, b = c / u.A;
  return double(y[a + i * u.A + b * u.A * u.n]);
}

// W[c * p + j] = sum_i Y[i, c] Q[i, j];  Q column j = qt[j * ldq + i]
template <typename TY>
__global__ void __launch_bounds__(NT) w_kernel(const TY* __restrict__ y, Unfold u,
                                               const double* __restrict__ qt, int64_t ldq, int p,
                                               double* __restrict__ wt) {
  __shared__ double Qs[TR * LQ];  // reused for the cross-warp reduction
  __shared__ double Ys[TR * CB];
  double* red = Qs;
  static_assert(8 * CB * kMaxP <= TR * LQ, "reduction must fit the Q tile");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = int64_t(blockIdx.x) * CB;
  const int ncb = u.cols - c0 < CB ? int(u.cols - c0) : CB;
  const bool two = p > 32;
  double acc[CB][2];
#pragma unroll
  for (int cb = 0; cb < CB; ++cb) acc[cb][0] = acc[cb][1] = 0.0;
  for (int64_t i0 = 0; i0 < u.n; i0 += TR) {
    const int rows = u.n - i0 < TR ? int(u.n - i0) : TR;
    for (int e = tid; e < p * TR; e += NT) {  // coalesced along i
      const int j = e / TR, ii = e % TR;
      Qs[ii * LQ + j] = ii < rows ? qt[int64_t(j) * ldq + i0 + ii] : 0.0;
    }
    if (u.A == 1) {  // mode 0: the unfolding is column-major, contiguous along i
      for (int e = tid; e < TR * CB; e += NT) {
        const int ii = e % TR, cb = e / TR;
        Ys[ii * CB + cb] = (ii < rows && cb < ncb) ? yat(y, u, i0 + ii, c0 + cb) : 0.0;
      }
    } else {         // contiguous along the column index
      for (int e = tid; e < TR * CB; e += NT) {
        const int cb = e % CB, ii = e / CB;
        Ys[ii * CB + cb] = (ii < rows && cb < ncb) ? yat(y, u, i0 + ii, c0 + cb) : 0.0;
      }
    }
    __syncthreads();
#pragma unroll 2
    for (int r = 0; r < TR / 8; ++r) {
      const int ii = warp * (TR / 8) + r;
      const double q0 = Qs[ii * LQ + lane];
      const double q1 = two ? Qs[ii * LQ + lane + 32] : 0.0;
#pragma unroll
      for (int cb = 0; cb < CB; ++cb) {
        const double yv = Ys[ii * CB + cb];
        acc[cb][0] = fma(yv, q0, acc[cb][0]);
        acc[cb][1] = fma(yv, q1, acc[cb][1]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int cb = 0; cb < CB; ++cb) {
    red[(warp * CB + cb) * kMaxP + lane] = acc[cb][0];
    red[(warp * CB + cb) * kMaxP + lane + 32] = acc[cb][1];
  }
  __syncthreads();
  for (int e = tid; e < ncb * p; e += NT) {  // fixed warp order
    const int cb = e / p, j = e % p;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[(w * CB + cb) * kMaxP + j];
    wt[(c0 + cb) * p + j] = s;
  }
}

// Z[i, j] = sum_c Y[i, c] W[c, j], written transposed: zt[j * ldz + i].
// grid = (ceil(n / RB), S); ws = S * tiles * RB * p doubles; cnt = tiles
// counters (zero before the first launch, left zero by every launch).
template <typename TY>
__global__ void __launch_bounds__(NT) z_kernel(const TY* __restrict__ y, Unfold u,
                                               const double* __restrict__ wt, int p,
                                               int64_t kper, double* __restrict__ zt,
                                               int64_t ldz, double* __restrict__ ws,
                                               unsigned* __restrict__ cnt) {
  __shared__ double Ws[TZ * LQ];
  __shared__ double Ys[RB * (TZ + 1)];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x, split = blockIdx.y, S = gridDim.y;
  const int64_t r0 = int64_t(tile) * RB;
  const int nrows = u.n - r0 < RB ? int(u.n - r0) : RB;
  const int64_t kb = int64_t(split) * kper;
  const int64_t ke = kb + kper < u.cols ? kb + kper : u.cols;
  const bool two = p > 32;
  double acc[4][2];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) acc[rr][0] = acc[rr][1] = 0.0;
  for (int64_t k0 = kb; k0 < ke; k0 += TZ) {
    const int kn = ke - k0 < TZ ? int(ke - k0) : TZ;
    for (int e = tid; e < TZ * p; e += NT) {  // W rows: coalesced along j
      const int cc = e / p, j = e % p;
      Ws[cc * LQ + j] = cc < kn ? wt[(k0 + cc) * p + j] : 0.0;
    }
    if (u.A == 1) {
      for (int e = tid; e < RB * TZ; e += NT) {
        const int rr = e % RB, cc = e / RB;
        Ys[rr * (TZ + 1) + cc] = (rr < nrows && cc < kn) ? yat(y, u, r0 + rr, k0 + cc) : 0.0;
      }
    } else {
      for (int e = tid; e < RB * TZ; e += NT) {
        const int cc = e % TZ, rr = e / TZ;
        Ys[rr * (TZ + 1) + cc] = (rr < nrows && cc < kn) ? yat(y, u, r0 + rr, k0 + cc) : 0.0;
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int cc = 0; cc < TZ; ++cc) {
      const double w0 = Ws[cc * LQ + lane];
      const double w1 = two ? Ws[cc * LQ + lane + 32] : 0.0;
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const double yv = Ys[(warp * 4 + rr) * (TZ + 1) + cc];
        acc[rr][0] = fma(yv, w0, acc[rr][0]);
        acc[rr][1] = fma(yv, w1, acc[rr][1]);
      }
    }
    __syncthreads();
  }
  if (S == 1) {
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int row = warp * 4 + rr;
      if (row >= nrows) continue;
      if (lane < p) zt[int64_t(lane) * ldz + r0 + row] = acc[rr][0];
      if (two && lane + 32 < p) zt[int64_t(lane + 32) * ldz + r0 + row] = acc[rr][1];
    }
    return;
  }
  const int ntiles = gridDim.x;
  double* part = ws + (int64_t(split) * ntiles + tile) * RB * kMaxP;
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    part[(warp * 4 + rr) * kMaxP + lane] = acc[rr][0];
    part[(warp * 4 + rr) * kMaxP + lane + 32] = acc[rr][1];
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned t = atomicAdd(cnt + tile, 1u);
    s_last = t == unsigned(S - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int e = tid; e < nrows * p; e += NT) {  // coalesced along i on the store
    const int row = e % nrows, j = e / nrows;
    double s = 0.0;
    for (int sp = 0; sp < S; ++sp)
      s += __ldcg(ws + (int64_t(sp) * ntiles + tile) * RB * kMaxP + row * kMaxP + j);
    zt[int64_t(j) * ldz + r0 + row] = s;
  }
  if (tid == 0) cnt[tile] = 0u;  // ready for the next launch / graph replay
}

// workspace layout (doubles): W [cols * p] | partials [S * tiles * RB * kMaxP]
// | Z [p * n] | counters [tiles] (unsigned)
struct Plan {
  int64_t tiles, splits, kper;
  int64_t w_off, part_off, z_off, cnt_off_bytes, bytes;
};

inline Plan plan(int64_t n, int64_t cols, int p) {
  Plan pl;
  pl.tiles = ceil_div(n, RB);
  // ~128 CTAs; each split at least TR columns
  int64_t s = ceil_div(128, pl.tiles);
  const int64_t smax = ceil_div(cols, TZ);
  if (s > smax) s = smax;
  if (s < 1) s = 1;
  pl.kper = ceil_div(ceil_div(cols, s), TZ) * TZ;
  pl.splits = ceil_div(cols, pl.kper);
  pl.w_off = 0;
  pl.part_off = cols * p;
  pl.z_off = pl.part_off + (pl.splits > 1 ? pl.splits * pl.tiles * RB * kMaxP : 0);
  pl.cnt_off_bytes = (pl.z_off + int64_t(p) * n) * 8;
  pl.bytes = pl.cnt_off_bytes + pl.tiles * 4;
  return pl;
}

}  // namespace gapply
}  // namespace sbt

namespace sbt {
namespace gapply {

// out[0] = ||x|| (fp64 sum of squares in a fixed order: one CTA, per-thread
// strided partials, tree reduction), out[1 + f] = flags[f]: the HOOI
// iteration's one device->host read (||G|| for the fit, the factors'
// convergence flags), replacing torch glue inside the captured iteration.
template <typename T>
__global__ void __launch_bounds__(1024) status_kernel(const T* __restrict__ x, int64_t count,
                                                      const int* __restrict__ flags, int nflags,
                                                      double* __restrict__ out) {
  __shared__ double red[32];
  const int tid = threadIdx.x;
  double s = 0.0;
  for (int64_t e = tid; e < count; e += blockDim.x) {
    const double v = double(x[e]);
    s = fma(v, v, s);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((tid & 31) == 0) red[tid >> 5] = s;
  __syncthreads();
  if (tid < 32) {
    s = tid < int(blockDim.x >> 5) ? red[tid] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (tid == 0) out[0] = sqrt(s);
  }
  if (tid < nflags) out[1 + tid] = double(flags[tid]);
}

}  // namespace gapply
}  // namespace sbt
