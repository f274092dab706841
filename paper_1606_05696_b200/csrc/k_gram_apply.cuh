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
#include <cooperative_groups.h>

#include "sbt_common.cuh"
#include "sm100_ptx.cuh"

namespace sbt {
namespace gapply {

constexpr int NT = 512;         // 16 warps: short per-warp instruction streams
constexpr int NWARP = NT / 32;
constexpr int kMaxP = 64;       // basis width
constexpr int CB = 8;           // W columns per CTA (one DMMA row tile)
constexpr int RB = 32;          // Z rows per CTA (2 per warp)

struct Unfold {
  int64_t n;     // rows (d_r)
  int64_t cols;  // prod of the other extents
  int64_t A;     // prod(d_<r): unit-stride run of a column index
};

// element offset of column c of the unfolding (row 0); row i adds i * A
// (32-bit division when the column index fits: 64-bit division is a long
// software sequence)
__device__ __forceinline__ int64_t col_base(const Unfold& u, int64_t c) {
  if (c < (int64_t(1) << 31)) {
    const uint32_t a = uint32_t(u.A), cc = uint32_t(c);
    const uint32_t q = cc / a;
    return int64_t(cc - q * a) + int64_t(q) * u.A * u.n;
  }
  return (c % u.A) + (c / u.A) * u.A * u.n;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Sum v[k] (k < NOUT, NOUT | 32) over the 32 lanes (fixed order): afterwards
// lane l holds the total of output l % NOUT.  32 / NOUT - 1 ... full butterfly
// steps first, then a reduce-scatter over NOUT lanes (31 shuffles in all).
template <int NOUT>
__device__ __forceinline__ double lane_reduce_scatter(double (&v)[NOUT], int lane) {
#pragma unroll
  for (int s = 16; s >= NOUT; s >>= 1)
#pragma unroll
    for (int k = 0; k < NOUT; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], s);
#pragma unroll
  for (int s = NOUT / 2; s >= 1; s >>= 1) {
    const bool up = lane & s;
#pragma unroll
    for (int k = 0; k < s; ++k) {
      const double keep = up ? v[k + s] : v[k];
      const double give = up ? v[k] : v[k + s];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, give, s);
    }
  }
  return v[0];
}

__device__ __forceinline__ void dmma8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// ---- W = Y_(r)^T Q ----------------------------------------------------------
// fp64 throughput per SM is ~250 GFLOP/s, so the product is spread over ~128
// CTAs of CB = 8 unfolding columns (one DMMA row tile); the 16 warps split
// the reduction (k-steps w, w + 16, ...) with one accumulator chain per 8-wide
// N tile (4 independent chains at p = 32) and are summed in warp order
// through shared memory.  Rows are staged in chunks of rch (a multiple of
// 32, chosen to fill <= ~200 KB; one chunk for n <= 768 at p = 32): Q rows
// and (mode 0) Y columns by 1-D TMA bulk copies issued one per lane across
// two warps on one mbarrier; other unfoldings by batched coalesced loads.
// Row padding (+4 elements) makes the DMMA fragment loads conflict-free.
constexpr int W_SMEM_MAX = 200 * 1024;
#ifdef SBT_RITZ_CLOCK
__device__ long long g_ga_clock[8];   // diagnostics build: CTA 0 thread 0 stamps
__device__ long long g_gz_clock[8];
#define GZ_STAMP(k) \
  do { if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) g_gz_clock[k] = clock64() - gz_t0; } while (0)
#define GA_STAMP(k) \
  do { if (threadIdx.x == 0 && blockIdx.x == 0) g_ga_clock[k] = clock64() - ga_t0; } while (0)
#else
#define GA_STAMP(k) do { } while (0)
#define GZ_STAMP(k) do { } while (0)
#endif
inline int w_rows_per_chunk(int64_t n, int p, int ysize) {
  const int64_t per = int64_t((p + 7) & ~7) * 8 + int64_t(CB) * ysize;  // bytes per ld unit
  int64_t r = W_SMEM_MAX / per - 4;
  r &= ~int64_t(31);
  const int64_t n32 = (n + 31) & ~int64_t(31);
  return int(n32 < r ? n32 : r);
}
inline int64_t w_smem_bytes(int rch, int p, int ysize) {
  const int64_t stage = (int64_t((p + 7) & ~7) * 8 + int64_t(CB) * ysize) * (rch + 4);
  const int64_t red = int64_t(NWARP) * 8 * kMaxP * 8;   // cross-warp partial tiles
  return stage > red ? stage : red;
}

// W[c * p + j] = sum_i Y[i, c] Q[i, j];  Q column j = qt[j * ldq + i].
// MODE_OUT: the same sums written as the packed mode-r product Y x_r Q^T
// (extent p at mode r): out[(c % A) + j * A + (c / A) * A * p], in TO.
// flags: bit 0 = Q rows by bulk copy (qt 16 B aligned, ldq and n even), bit 1 =
// Y columns by bulk copy (mode 0, 16 B aligned columns).
template <typename TY, typename TO, bool MODE_OUT>
__global__ void __launch_bounds__(NT) w_kernel(const TY* __restrict__ y, Unfold u,
                                               const double* __restrict__ qt, int64_t ldq, int p,
                                               TO* __restrict__ wt, int rch, int flags) {
  extern __shared__ __align__(16) unsigned char smw_raw[];
#ifdef SBT_RITZ_CLOCK
  const long long ga_t0 = clock64();
#endif
  const int ld = rch + 4;
  const int ntn = (p + 7) >> 3;              // 8-wide N tiles (<= 8)
  double* Qs = reinterpret_cast<double*>(smw_raw);             // [8 ntn][ld]
  TY* Ys = reinterpret_cast<TY*>(Qs + int64_t(8 * ntn) * ld);   // [CB][ld]
  __shared__ int64_t s_col[CB];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = int64_t(blockIdx.x) * CB;
  const int ncb = u.cols - c0 < CB ? int(u.cols - c0) : CB;
  const int A = int(u.A);
  const int fr = lane >> 2, fk = lane & 3;
  const bool qbulk = flags & 1, ybulk = flags & 2;
  if (tid < CB) s_col[tid] = col_base(u, c0 + (tid < ncb ? tid : 0));
  if (tid == 0) {
    ptx::mbar_init(&bar, 2);                 // one arrival per issuing warp
    ptx::fence_mbarrier_init();
  }
  double acc[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = 0.0;
  __syncthreads();
  GA_STAMP(0);
  int chunk = 0;
  for (int64_t i0 = 0; i0 < u.n; i0 += rch, ++chunk) {
    const int rows = u.n - i0 < rch ? int(u.n - i0) : rch;
    const int rows4 = (rows + 3) & ~3;
    if (qbulk || ybulk) {
      // warp 0: the p basis rows; warp 1: the ncb Y columns; lane-parallel issue
      if (warp == 0) {
        if (lane == 0) {
          ptx::fence_proxy_async_smem();     // the previous chunk's reads precede these writes
          ptx::mbar_arrive_expect_tx(&bar, qbulk ? uint32_t(p) * rows * 8 : 0u);
        }
        __syncwarp();
        if (qbulk)
          for (int j = lane; j < p; j += 32)
            ptx::bulk_load(Qs + int64_t(j) * ld, qt + int64_t(j) * ldq + i0, uint32_t(rows) * 8,
                           &bar);
      } else if (warp == 1) {
        if (lane == 0) {
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive_expect_tx(&bar, ybulk ? uint32_t(ncb) * rows * uint32_t(sizeof(TY)) : 0u);
        }
        __syncwarp();
        if (ybulk && lane < ncb)
          ptx::bulk_load(Ys + int64_t(lane) * ld, y + s_col[lane] + i0,
                         uint32_t(rows) * uint32_t(sizeof(TY)), &bar);
      }
    }
    // zero padding (only when needed): rows [rows, rows4), rows past p / ncb
    if (rows4 != rows || (p & 7))
      for (int j = 0; j < 8 * ntn; ++j)
        for (int k = (j < p ? rows : 0) + tid; k < rows4; k += NT) Qs[int64_t(j) * ld + k] = 0.0;
    if (rows4 != rows || ncb < CB)
      for (int cb = 0; cb < CB; ++cb)
        for (int k = (cb < ncb ? rows : 0) + tid; k < rows4; k += NT) Ys[int64_t(cb) * ld + k] = TY(0);
    if (!qbulk) {
      for (int j = 0; j < p; ++j)
        for (int ii = tid; ii < rows; ii += NT) Qs[int64_t(j) * ld + ii] = qt[int64_t(j) * ldq + i0 + ii];
    }
    if (!ybulk) {
      if (A == 1) {
        for (int ii = tid; ii < rows; ii += NT) {
          TY v[CB];
#pragma unroll
          for (int cb = 0; cb < CB; ++cb) v[cb] = cb < ncb ? y[s_col[cb] + i0 + ii] : TY(0);
#pragma unroll
          for (int cb = 0; cb < CB; ++cb)
            if (cb < ncb) Ys[int64_t(cb) * ld + ii] = v[cb];
        }
      } else {                                // contiguous along the columns
        constexpr int YB = 8, RS = NT / CB;   // RS rows per pass
        const int cb = tid & (CB - 1);
        const TY* src = y + s_col[cb] + i0 * A;
        for (int ib = tid / CB; ib < rows; ib += YB * RS) {
          TY v[YB];
#pragma unroll
          for (int t = 0; t < YB; ++t) {
            const int ii = ib + t * RS;
            v[t] = (cb < ncb && ii < rows) ? src[int64_t(ii) * A] : TY(0);
          }
#pragma unroll
          for (int t = 0; t < YB; ++t) {
            const int ii = ib + t * RS;
            if (cb < ncb && ii < rows) Ys[int64_t(cb) * ld + ii] = v[t];
          }
        }
      }
    }
    GA_STAMP(1);
    if (qbulk || ybulk) ptx::mbar_wait(&bar, uint32_t(chunk & 1));
    GA_STAMP(2);
    __syncthreads();
    GA_STAMP(3);
    const TY* ya = Ys + int64_t(fr) * ld + fk;
    for (int k = 4 * warp; k < rows4; k += 4 * NWARP) {
      const double a = double(ya[k]);
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (t < ntn) dmma8x8x4(acc[t], a, Qs[int64_t(8 * t + fr) * ld + fk + k]);
    }
    GA_STAMP(4);
    __syncthreads();
  }
  // cross-warp sum in warp order: partial tiles through shared memory
  double* red = reinterpret_cast<double*>(smw_raw);   // [NWARP][8][kMaxP]
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if (t >= ntn) break;
    red[(warp * 8 + fr) * kMaxP + 8 * t + 2 * fk] = acc[t][0];
    red[(warp * 8 + fr) * kMaxP + 8 * t + 2 * fk + 1] = acc[t][1];
  }
  __syncthreads();
  for (int e = tid; e < CB * p; e += NT) {
    const int cb = e / p, j = e % p;
    if (cb >= ncb) continue;
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) sum += red[(w * 8 + cb) * kMaxP + j];
    const int64_t c = c0 + cb;
    if (MODE_OUT) wt[(c % u.A) + int64_t(j) * u.A + (c / u.A) * u.A * p] = TO(sum);
    else wt[c * p + j] = TO(sum);
  }
  GA_STAMP(5);
}

// ---- Z = Y_(r) W ---------------------------------------------------------------
// Z[i, j] = sum_c Y[i, c] W[c, j], written transposed: zt[j * ldz + i].
// grid = (ceil(n / RB), ZS): a cluster of ZS CTAs per RB-row tile, CTA s of
// the cluster reducing columns [s kper, (s + 1) kper) in chunks of KZ with
// everything a chunk reads requested at once; the ZS partial tiles are summed
// in split order through distributed shared memory (each CTA one slice of the
// outputs) -- deterministic, no global workspace, no atomics.
constexpr int ZS = 8;
constexpr int KZ = 128;
constexpr int LDY = KZ + 4;             // padded rows: conflict-free fragments
constexpr int LDW = kMaxP + 8;          // rows 8 doubles apart in the banks
constexpr int Z_SMEM_BYTES = KZ * LDW * 8 + RB * LDY * 8 + KZ * 8;
static_assert(RB * kMaxP <= KZ * LDW, "partial tile fits the W area");
template <typename TY>
__global__ void __cluster_dims__(1, ZS, 1) __launch_bounds__(NT)
z_kernel(const TY* __restrict__ y, Unfold u, const double* __restrict__ wt, int p, int64_t kper,
         double* __restrict__ zt, int64_t ldz) {
  extern __shared__ __align__(16) double smz[];
#ifdef SBT_RITZ_CLOCK
  const long long gz_t0 = clock64();
#endif
  double* Ws = smz;                                // [KZ][LDW]  (row = column c of Y)
  double* Ys = smz + KZ * LDW;                     // [RB][LDY]
  int64_t* colb = reinterpret_cast<int64_t*>(Ys + RB * LDY);  // [KZ]
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x, split = blockIdx.y;
  const int64_t r0 = int64_t(tile) * RB;
  const int nrows = u.n - r0 < RB ? int(u.n - r0) : RB;
  const int64_t kb = int64_t(split) * kper;
  const int64_t ke = kb + kper < u.cols ? kb + kper : u.cols;
  const int A = int(u.A);
  const int fr = lane >> 2, fk = lane & 3;
  const int ntn = (p + 7) >> 3;
  const int ntiles_out = (RB / 8) * ntn;             // <= 32: at most 2 per warp
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int64_t k0 = kb; k0 < ke; k0 += KZ) {
    const int kn = int(ke - k0 < KZ ? ke - k0 : KZ);
    const int kn4 = (kn + 3) & ~3;
    // W rows: p doubles each, 16-byte async copies into padded rows
    const double* src = wt + k0 * p;
    const int pc = (p + 1) >> 1;                     // 16-byte chunks per row
    const bool even = (p & 1) == 0;
    for (int e = tid; e < kn4 * pc; e += NT) {
      const int cc = e / pc, h = e % pc;
      double* dst = Ws + cc * LDW + 2 * h;
      if (cc < kn && even) cp_async16(dst, src + int64_t(cc) * p + 2 * h);
      else {
        dst[0] = cc < kn ? src[int64_t(cc) * p + 2 * h] : 0.0;
        dst[1] = (cc < kn && 2 * h + 1 < p) ? src[int64_t(cc) * p + 2 * h + 1] : 0.0;
      }
    }
    for (int e = tid; e < kn4 * (8 * ntn - p); e += NT) {  // zero the N-tile padding
      const int cc = e / (8 * ntn - p), j = p + e % (8 * ntn - p);
      Ws[cc * LDW + j] = 0.0;
    }
    if (tid < KZ) colb[tid] = tid < kn ? col_base(u, k0 + tid) + r0 * A : 0;
    __syncthreads();
    GZ_STAMP(0);
    {                   // all RB x KZ loads in flight, then the stores
      constexpr int YPT = RB * KZ / NT;
      double v[YPT];
#pragma unroll
      for (int t = 0; t < YPT; ++t) {
        const int e = tid + t * NT;
        int rr, cc;
        if (A == 1) { rr = e & (RB - 1); cc = e / RB; }   // contiguous along the rows
        else        { cc = e & (KZ - 1); rr = e / KZ; }   // contiguous along the columns
        v[t] = (rr < nrows && cc < kn) ? double(y[colb[cc] + int64_t(rr) * A]) : 0.0;
      }
#pragma unroll
      for (int t = 0; t < YPT; ++t) {
        const int e = tid + t * NT;
        int rr, cc;
        if (A == 1) { rr = e & (RB - 1); cc = e / RB; }
        else        { cc = e & (KZ - 1); rr = e / KZ; }
        Ys[rr * LDY + cc] = v[t];
      }
    }
    GZ_STAMP(1);
    cp_async_wait_all();
    __syncthreads();
    GZ_STAMP(2);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int ot = warp + q * NWARP;
      if (ot >= ntiles_out) break;
      const int mt = ot % (RB / 8), nt = ot / (RB / 8);
      const double* ya = Ys + (8 * mt + fr) * LDY + fk;
      const double* wb = Ws + fk * LDW + 8 * nt + fr;
      double a4[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};  // k-step chains
      int k = 0;
      for (; k + 12 < kn4; k += 16) {
#pragma unroll
        for (int c = 0; c < 4; ++c) dmma8x8x4(a4[c], ya[k + 4 * c], wb[(k + 4 * c) * LDW]);
      }
#pragma unroll
      for (int c = 0; c < 3; ++c)          // tail: at most 3 steps
        if (k + 4 * c < kn4) dmma8x8x4(a4[c], ya[k + 4 * c], wb[(k + 4 * c) * LDW]);
#pragma unroll
      for (int h = 0; h < 2; ++h) acc[q][h] += (a4[0][h] + a4[1][h]) + (a4[2][h] + a4[3][h]);
    }
    __syncthreads();
  }
  // partial tile [RB][kMaxP] in this CTA's W area, then the cluster sums
  double* part = Ws;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int ot = warp + q * NWARP;
    if (ot >= ntiles_out) break;
    const int mt = ot % (RB / 8), nt = ot / (RB / 8);
#pragma unroll
    for (int h = 0; h < 2; ++h) part[(8 * mt + fr) * kMaxP + 8 * nt + 2 * fk + h] = acc[q][h];
  }
  GZ_STAMP(3);
  cluster.sync();
  GZ_STAMP(4);
  const int crank = int(cluster.block_rank());
  const int nout = nrows * p, per = (nout + ZS - 1) / ZS;
  // 4 threads per output (2 splits each), pairs then quads summed by shuffles:
  // ((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7)), a fixed order
  static_assert(ZS == 8, "4 lanes x 2 splits");
  const int sub = tid & 3;
  for (int e0 = crank * per; e0 < (crank + 1) * per && e0 < nout; e0 += NT / 4) {
    const int e = e0 + (tid >> 2);
    const bool ok = e < (crank + 1) * per && e < nout;
    const int row = ok ? e % nrows : 0, j = ok ? e / nrows : 0;   // stores coalesced along i
    const double* a = part + row * kMaxP + j;
    double v = *cluster.map_shared_rank(a, 2 * sub) + *cluster.map_shared_rank(a, 2 * sub + 1);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    if (ok && sub == 0) zt[int64_t(j) * ldz + r0 + row] = v;
  }
  GZ_STAMP(5);
  cluster.sync();   // no CTA exits while its partial may still be read
  GZ_STAMP(6);
}

// workspace layout (doubles): W [cols * p] | Z [p * n]
struct Plan {
  int64_t tiles, kper;
  int64_t w_off, z_off, bytes;
};

inline Plan plan(int64_t n, int64_t cols, int p) {
  Plan pl;
  pl.tiles = ceil_div(n, RB);
  pl.kper = ceil_div(ceil_div(cols, ZS), 4) * 4;
  pl.w_off = 0;
  pl.z_off = cols * p;
  pl.bytes = (pl.z_off + int64_t(p) * n) * 8;
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
  const int64_t step = int64_t(blockDim.x) * 8;
  for (int64_t e0 = tid; e0 < count; e0 += step) {  // 8 loads in flight per thread
    double v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int64_t e = e0 + int64_t(t) * blockDim.x;
      v[t] = e < count ? double(x[e]) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) s = fma(v[t], v[t], s);
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
