// Rayleigh-Ritz step of the HOOI eigensolver, entirely on the device.
//
// The reference takes the leading `rank` eigenvectors of each mode's Gram
// matrix (tucker.py:63-76, Jacobi on the full n x n Gram, tucker.py:21-60).
// HOOI here runs warm-started subspace sweeps per factor (tucker.py
// top_eigh): Q = previous factor (n x p), Z = G Q.  This kernel finishes a
// sweep without a host round trip, so a whole HOOI iteration is launch-only.
// One 8-CTA cluster:
//   * H = Q^T Z (p x p): each CTA sums its row tiles of Q and Z, the partials
//     are added in CTA order through distributed shared memory (or H comes
//     from the caller's m = [Q Z]^T Z);
//   * CTA 0 diagonalises H: Newton refinement for a warm start (A = V^T H V,
//     V <- V (I + E) with E_ij = A_ij / (A_jj - A_ii), re-orthonormalised by
//     one Newton-Schulz step; quadratic convergence in a few 32 x 32 products),
//     then cyclic Jacobi for whatever is left (round-robin pairing: a step is
//     A <- J^T A J with J a product of disjoint rotations; each 2 x 2 block of
//     A and V is updated by one thread, one barrier per step);
//   * eigenvalues sorted descending;
//   * all CTAs: U = Q V, Y = Z V (= G U) for the leading `rank` Ritz vectors
//     from row tiles of Q and Z staged in shared memory; residuals
//     ||Y_j - w_j U_j|| and the convergence flag max_j ||.|| <= tol * w_max
//     (the same test as top_eigh);
//   * sign rule of tucker.py:71-75 (largest |entry| of each column positive,
//     first index on ties), combined across the cluster; optional fp32 copy.
// p <= kMaxP.  The caller checks `flag` later (once per iteration) and redoes
// the iteration on the host path if any factor did not converge.
#pragma once
#include <cooperative_groups.h>

#include "sbt_common.cuh"

namespace sbt {
namespace ritz {

#ifdef SBT_RITZ_CLOCK
// [0..11]: CTA 0 thread 0 cycles since kernel start at the STAMP points;
// [15]: cycles of the Jacobi steps
__device__ long long g_ritz_clock[24];
#define RITZ_STAMP(k) \
  do { if (tid == 0 && crank == 0) g_ritz_clock[k] = clock64() - t_start; } while (0)
#else
#define RITZ_STAMP(k) do { } while (0)
#endif
constexpr int kMaxP = 64;
constexpr int kHalf = kMaxP / 2;
constexpr int kThreads = 512;
constexpr int kCluster = 8;                    // CTAs sharing the Ritz-vector phase
constexpr int LDS = kMaxP + 4;                 // 8-word row skew: conflict-free DMMA row fragments
constexpr int MAT = kMaxP * LDS;               // one P x P matrix (padded rows)
constexpr int kTileRows = 64;                  // Q / Z row tile
constexpr int LDT = kTileRows + 4;             // tile row stride (conflict-free DMMA fragments)
constexpr int REGION0 = 5 * MAT;  // >= the two Q / Z tiles (2 * kMaxP * LDT)
static_assert(2 * kMaxP * LDT <= 2 * MAT, "Q / Z tiles fill slots 0-1; U / Y tiles use 2-3");
constexpr int kTri = kHalf * (kHalf + 1) / 2;  // upper-triangular 2 x 2 blocks
constexpr int SMEM_BYTES =
    (REGION0 + 4 * kMaxP) * 8 + (2 * kMaxP) * 4 + (kMaxP * kMaxP + 2 * kTri) + 64;

// C = op(X) Y for P x P matrices in shared memory (row stride LDS), 2 x 2
// register blocks per thread; EPI 1 stores 1.5 I - 0.5 C (Newton-Schulz).
template <bool TX, int EPI>
__device__ __forceinline__ void small_mm_unused(const double* X, const double* Y, double* C, int P,
                                         int tid) {
  const int hb = P / 2;
  for (int blk = tid; blk < hb * hb; blk += kThreads) {
    const int i0 = 2 * (blk / hb), j0 = 2 * (blk % hb);
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
    for (int l = 0; l < P; ++l) {
      const double x0 = TX ? X[l * LDS + i0] : X[i0 * LDS + l];
      const double x1 = TX ? X[l * LDS + i0 + 1] : X[(i0 + 1) * LDS + l];
      const double y0 = Y[l * LDS + j0], y1 = Y[l * LDS + j0 + 1];
      c00 = fma(x0, y0, c00);
      c01 = fma(x0, y1, c01);
      c10 = fma(x1, y0, c10);
      c11 = fma(x1, y1, c11);
    }
    if (EPI == 1) {
      c00 = (i0 == j0 ? 1.5 : 0.0) - 0.5 * c00;
      c01 = -0.5 * c01;
      c10 = -0.5 * c10;
      c11 = (i0 == j0 ? 1.5 : 0.0) - 0.5 * c11;
    }
    C[i0 * LDS + j0] = c00;
    C[i0 * LDS + j0 + 1] = c01;
    C[(i0 + 1) * LDS + j0] = c10;
    C[(i0 + 1) * LDS + j0 + 1] = c11;
  }
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// C = op(X) Y for P x P matrices in shared memory (row stride LDS) on the
// fp64 tensor pipe: 8 x 8 DMMA output tiles over the 16 warps, two
// accumulator chains per tile (even / odd k-steps, summed at the end: a fixed
// order); k >= P reads as zero, rows / columns >= P are not stored.  EPI 1
// stores 1.5 I - 0.5 C (Newton-Schulz).  All threads of the CTA call it.
// One out-of-line copy (runtime TX / EPI): the serial eigen phase runs each
// code path a few times only, so instruction-cache misses on cold inlined
// copies cost more than the arithmetic.
__device__ __noinline__ void dmma_mm_rt(const double* X, const double* Y, double* C, int P,
                                        int tid, bool TX, int EPI) {
  const int warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fk = lane & 3;
  const int nt = (P + 7) >> 3;
  for (int t = warp; t < nt * nt; t += kThreads / 32) {
    const int mt = t / nt, ntl = t % nt;
    const int m = 8 * mt + fr, n = 8 * ntl + fr;
    // k-step s accumulates into chain s % 8: the fp64 tensor pipe's long
    // dependent-issue latency would otherwise serialise the P / 4 steps
    double c[8][2];
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
    for (int k0 = 0; k0 < P; k0 += 32) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = k0 + 4 * q + fk;
        const double a = k < P ? (TX ? X[k * LDS + m] : X[m * LDS + k]) : 0.0;
        const double b = k < P ? Y[k * LDS + n] : 0.0;
        dmma(c[q], a, b);
      }
    }
    double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 8; ++q) c0[0] += c[q][0], c0[1] += c[q][1];
    const int row = 8 * mt + fr;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = 8 * ntl + 2 * fk + h;
      if (row < P && col < P) {
        const double v = c0[h] + c1[h];
        C[row * LDS + col] = EPI == 1 ? (row == col ? 1.5 : 0.0) - 0.5 * v : v;
      }
    }
  }
}

// q / z: the columns of Q and of Z = G Q as p rows each (row j at q + j * ldq,
// z + j * ldz; the entry point's qz = [Q | Z] is q = qz, z = qz + p * n);
// m: the (2p x p) column-major product [Q Z]^T Z (ld 2p).
// m == nullptr: H = Q^T Z is formed in-kernel.
// ut: rank rows of length n (U column-major); yt (optional): the same for
// Y = G U (the next sweep's basis, before the sign rule); ut32 (optional): U
// rounded to fp32; w: rank eigenvalues
// (descending); flag[0] = converged; rel[0] = max residual / w_max,
// rel[1] = Jacobi sweeps, rel[2..4] = SM cycles of the eigen / Ritz-vector /
// sign phases, rel[5] = Newton refinement steps (diagnostics).
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads, 1)
ritz_kernel(const double* __restrict__ q, int64_t ldq, const double* __restrict__ z,
            int64_t ldz, const double* __restrict__ m, int64_t n, int p,
            int rank, double tol, double* __restrict__ ut, double* __restrict__ yt,
            float* __restrict__ ut32, double* __restrict__ w, int* __restrict__ flag,
            double* __restrict__ rel) {
  extern __shared__ __align__(16) double smr[];
  // eigen phase: A double-buffered at smr + {0, 1} * MAT (buffer 1 is W in the
  // Newton phase), V at smr + 2 * MAT, H at smr + 3 * MAT, S at smr + 4 * MAT
  double* V = smr + 2 * MAT;
  double* H = smr + 3 * MAT;
  double* S = smr + 4 * MAT;
  double* W = smr + MAT;
  double* Qs = smr;                     // [p][LDT] row tiles (reuse A / V)
  double* Zs = smr + kMaxP * LDT;
  double* Us = smr + 2 * MAT;           // Ritz phase: U / Y row tiles [64][LDS]
  double* Yv = smr + 3 * MAT;
  double* Vs = smr + 4 * MAT;           // [p][LDS]: sorted leading eigenvectors (reuses S)
  double* wv = smr + REGION0;           // sorted eigenvalues
  double* res = wv + kMaxP;             // [rank] squared residuals
  double* amax = res + kMaxP;           // [rank] max |U| per column
  double* sgn = amax + kMaxP;           // [rank] sign rule
  int* perm = reinterpret_cast<int*>(sgn + kMaxP);               // perm[j] = index of the j-th largest
  int* s_arg = perm + kMaxP;            // first row attaining amax
  unsigned char* pairs = reinterpret_cast<unsigned char*>(s_arg + kMaxP);  // [P-1][P]
  unsigned char* tri = pairs + kMaxP * kMaxP;                               // [kTri][2]
  __shared__ double s_red[2];
  __shared__ int s_clamp;
  const int tid = threadIdx.x;
  const long long t_start = clock64();
  const int P = p + (p & 1);            // even; a padding index is decoupled
  const int half = P / 2;
  const int ntri = half * (half + 1) / 2;
  const int nitems = ntri + half * half;  // A blocks (i <= j) + V blocks
  const int64_t ldm = 2 * int64_t(p);

  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = int(cluster.block_rank());
  int sweeps = 0, newton = 0;
  long long t_jacobi = t_start;
  // stage rows [i0, i0 + rows) of Q and Z into Qs / Zs ([l][LDT], row fastest)
  auto load_tile = [&](int64_t i0, int rows) {
    for (int e = tid; e < p * kTileRows; e += kThreads) {
      const int l = e / kTileRows, rr = e % kTileRows;
      const bool in = rr < rows;
      Qs[l * LDT + rr] = in ? q[int64_t(l) * ldq + i0 + rr] : 0.0;
      Zs[l * LDT + rr] = in ? z[int64_t(l) * ldz + i0 + rr] : 0.0;
    }
  };
  // m == nullptr: H = Q^T Z from the cluster's row tiles (partial per CTA in
  // slot 4, summed in CTA order by CTA 0) instead of a separate GEMM
  double* Hp = smr + 4 * MAT;
  if (m == nullptr) {
    // partial H = Q_t^T Z_t over this CTA's row tiles on the fp64 tensor pipe:
    // 8 x 8 output tiles over the 16 warps, accumulated across the tiles
    const int warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fk = lane & 3;
    const int nt = (p + 7) >> 3;
    double hacc[4][4][2];   // [tile][chain]: 4 independent k-step chains per tile
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < 4; ++c) hacc[q][c][0] = hacc[q][c][1] = 0.0;
    for (int64_t i0 = int64_t(crank) * kTileRows; i0 < n; i0 += kCluster * kTileRows) {
      const int rows = n - i0 < kTileRows ? int(n - i0) : kTileRows;
      load_tile(i0, rows);
      __syncthreads();
      RITZ_STAMP(0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int t = warp + 16 * q;
        if (t >= nt * nt) break;
        const double* qa = Qs + (8 * (t / nt) + fr) * LDT + fk;
        const double* zb = Zs + (8 * (t % nt) + fr) * LDT + fk;
#pragma unroll
        for (int r0 = 0; r0 < kTileRows; r0 += 16)
#pragma unroll
          for (int c = 0; c < 4; ++c) dmma(hacc[q][c], qa[r0 + 4 * c], zb[r0 + 4 * c]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = warp + 16 * q;
      if (t >= nt * nt) break;
      const int row = 8 * (t / nt) + fr;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = 8 * (t % nt) + 2 * fk + h;
        const double v = (hacc[q][0][h] + hacc[q][1][h]) + (hacc[q][2][h] + hacc[q][3][h]);
        if (row < p && col < p) Hp[row * LDS + col] = v;
      }
    }
    RITZ_STAMP(1);
    cluster.sync();
    // each CTA sums a slice of the entries over the cluster (CTA order, the
    // eight remote loads in flight together) into CTA 0's slot 3
    double* H0 = cluster.map_shared_rank(smr + 3 * MAT, 0);
    const int per = (p * p + kCluster - 1) / kCluster;
    for (int e = crank * per + tid; e < (crank + 1) * per && e < p * p; e += kThreads) {
      const int off = (e / p) * LDS + e % p;
      double v[kCluster];
#pragma unroll
      for (int c = 0; c < kCluster; ++c) v[c] = *cluster.map_shared_rank(Hp + off, c);
      double sum = 0.0;
#pragma unroll
      for (int c = 0; c < kCluster; ++c) sum += v[c];
      H0[off] = sum;
    }
    cluster.sync();
    RITZ_STAMP(2);
  }
  if (crank == 0) {  // the eigen phase runs on CTA 0; the others wait
    // round-robin schedule (circle method: position 0 holds player P-1) and
    // the upper-triangular block list
    for (int e = tid; e < (P - 1) * half; e += kThreads) {
      const int step = e / half, i = e % half;
      auto idx = [&](int pos) { return pos == 0 ? P - 1 : (pos - 1 + step) % (P - 1); };
      pairs[step * P + 2 * i] = (unsigned char)idx(i);
      pairs[step * P + 2 * i + 1] = (unsigned char)idx(P - 1 - i);
    }
    if (tid < half) {
      int base = tid * half - tid * (tid - 1) / 2;  // blocks (tid, tid..half-1)
      for (int j = tid; j < half; ++j, ++base) {
        tri[2 * base] = (unsigned char)tid;
        tri[2 * base + 1] = (unsigned char)j;
      }
    }
    if (tid < 2) s_red[tid] = 0.0;
    __syncthreads();
    double fro = 0.0;
    for (int e = tid; e < P * P; e += kThreads) {
      const int i = e / P, j = e % P;
      double h = 0.0;
      if (i < p && j < p) {
        if (m) {
          h = 0.5 * (m[i + j * ldm] + m[j + i * ldm]);
        } else {  // the cluster-summed Q^T Z (slot 3, read before H is written)
          h = 0.5 * (H[i * LDS + j] + H[j * LDS + i]);
        }
      }
      smr[i * LDS + j] = h;
      V[i * LDS + j] = i == j ? 1.0 : 0.0;
      fro += h * h;
    }
    for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
    if ((tid & 31) == 0) atomicAdd(&s_red[0], fro);
    __syncthreads();
    for (int e = tid; e < P * P; e += kThreads) {  // H keeps the symmetrised start
      const int i = e / P, j = e % P;
      H[i * LDS + j] = smr[i * LDS + j];
    }
    __syncthreads();
    // rotate only while |a_pq| > floor: an off-diagonal d left in H adds at
    // most ~d to a Ritz residual, which is tested against tol * w_max, so
    // d <= 0.01 tol ||H||_F (<= 0.06 tol w_max for p <= 32) changes no decision;
    // a warm start is often already there (a test relative to
    // sqrt(a_pp a_qq) would keep rotating rounding noise between the smallest
    // Ritz values)
// rotation / refinement floor as a fraction of tol: f leaves at most
// f tol ||H||_F <= f sqrt(p) tol w_max of off-diagonal in the Ritz residual
// test.  p <= 32: f = 0.05 (<= 0.28 tol w_max; measured on the 512^3 rank-32
// HOOI: 1e-2 -> 0.05 drops a Newton step, 0.496 -> 0.459 ms per iteration, no
// host redos, fit unchanged to 5e-8); wider bases keep f = 0.01
#ifndef SBT_RITZ_FLOOR
#define SBT_RITZ_FLOOR 0.05
#endif
    const double floor_frac = p <= 32 ? SBT_RITZ_FLOOR : 1e-2;
    const double floor_abs = fmax(1e-15, floor_frac * tol) * sqrt(s_red[0]);
    RITZ_STAMP(3);
    // rotation of pair (a, b) from the current A: J[a][a] = J[b][b] = c,
    // J[a][b] = s, J[b][a] = -s.  t = tan(angle) at float precision (any t
    // gives an orthogonal rotation; |th| <= 2e15 above the floor), c = (1 +
    // t^2)^-1/2 by two fp64 Newton steps from the float estimate.  Every
    // thread that needs a rotation computes it from the same inputs.
    auto rot = [&](const double* Ao, int a, int b, double& c, double& sn) {
      const double apq = Ao[a * LDS + b];
      c = 1.0;
      sn = 0.0;
      if (fabs(apq) > floor_abs) {
        const double app = Ao[a * LDS + a], aqq = Ao[b * LDS + b];
        const float th = __fdividef(float(aqq - app), float(2.0 * apq));
        const float tf = copysignf(1.f, th) / (fabsf(th) + sqrtf(fmaf(th, th, 1.f)));
        const double t = double(tf), v = fma(t, t, 1.0);
        double x = double(rsqrtf(float(v)));
        x = x * fma(-0.5 * v, x * x, 1.5);
        x = x * fma(-0.5 * v, x * x, 1.5);
        c = x;
        sn = t * x;
      }
    };
    // Newton refinement for a warm start (H nearly diagonal): with A = V^T H V,
    // V <- V (I + E), E_ij = A_ij / (A_jj - A_ii) (antisymmetric: annihilates
    // A's off-diagonal to first order), re-orthonormalised by one Newton-Schulz
    // step V <- W (1.5 I - 0.5 W^T W).  Quadratic convergence in a handful of
    // small matrix products instead of (p-1)-step Jacobi sweeps; pairs too
    // close for the first-order update (|A_ij| > |A_jj - A_ii| / 4) hand over
    // to the Jacobi sweeps below, which also finish anything left.
    for (int itn = 0; itn < 4; ++itn) {
      if (tid == 0) s_red[1] = 0.0, s_clamp = 0;
      __syncthreads();
      double off = 0.0;
      int clamp = 0;
      for (int e = tid; e < P * P; e += kThreads) {
        const int i = e / P, j = e % P;
        double x = 1.0;
        if (i != j) {
          const double a = smr[i * LDS + j], d = smr[j * LDS + j] - smr[i * LDS + i];
          off = fmax(off, fabs(a));
          x = 0.0;
          if (fabs(a) > floor_abs) {
            if (fabs(a) <= 0.25 * fabs(d)) x = a / d;
            else clamp = 1;
          }
        }
        S[i * LDS + j] = x;
      }
      for (int o = 16; o > 0; o >>= 1) {
        off = fmax(off, __shfl_xor_sync(0xffffffffu, off, o));
        clamp |= __shfl_xor_sync(0xffffffffu, clamp, o);
      }
      if ((tid & 31) == 0) {
        atomicMax(reinterpret_cast<unsigned long long*>(&s_red[1]), __double_as_longlong(off));
        if (clamp) atomicOr(&s_clamp, 1);
      }
      __syncthreads();
      if (itn == 0) RITZ_STAMP(16);
      if (s_red[1] <= floor_abs || s_clamp) break;
      ++newton;
      dmma_mm_rt(V, S, W, P, tid, false, 0);   // W = V (I + E)
      __syncthreads();
      if (itn == 0) RITZ_STAMP(17);
      dmma_mm_rt(W, W, S, P, tid, true, 1);    // S = 1.5 I - 0.5 W^T W
      __syncthreads();
      if (itn == 0) RITZ_STAMP(18);
      dmma_mm_rt(W, S, V, P, tid, false, 0);   // V = W S
      __syncthreads();
      dmma_mm_rt(H, V, W, P, tid, false, 0);   // W = H V
      __syncthreads();
      dmma_mm_rt(V, W, smr, P, tid, true, 0);  // A = V^T H V
      __syncthreads();
      if (itn == 0) RITZ_STAMP(19);
      for (int e = tid; e < P * P; e += kThreads) {
        const int i = e / P, j = e % P;
        if (i < j) {
          const double a = 0.5 * (smr[i * LDS + j] + smr[j * LDS + i]);
          smr[i * LDS + j] = a;
          smr[j * LDS + i] = a;
        }
      }
      __syncthreads();
      if (itn == 0) RITZ_STAMP(20);
    }
    RITZ_STAMP(4);
    int cur = 0;
    for (int sweep = 0; sweep < 40; ++sweep) {
      // converged when no off-diagonal element exceeds the floor
      const double* Ac = smr + cur * MAT;
      double off = 0.0;
      for (int e = tid; e < P * P; e += kThreads) {
        const int i = e / P, j = e % P;
        if (i != j) off = fmax(off, fabs(Ac[i * LDS + j]));
      }
      for (int o = 16; o > 0; o >>= 1) off = fmax(off, __shfl_xor_sync(0xffffffffu, off, o));
      if (tid == 0) s_red[1] = 0.0;
      __syncthreads();
      if ((tid & 31) == 0)
        atomicMax(reinterpret_cast<unsigned long long*>(&s_red[1]), __double_as_longlong(off));
      __syncthreads();
      if (s_red[1] <= floor_abs) break;
      ++sweeps;
      for (int step = 0; step < P - 1; ++step) {
  #ifdef SBT_RITZ_CLOCK
        const long long c0 = clock64();
  #endif
        // one barrier per step: rotations and blocks read A (buffer cur), the
        // new A goes to the other buffer; V is updated in place (each V block
        // belongs to one thread and V is not read by the rotations)
        const double* Ao = smr + cur * MAT;
        double* An = smr + (cur ^ 1) * MAT;
        const unsigned char* pr = pairs + step * P;
        for (int it = tid; it < nitems; it += kThreads) {
          if (it < ntri) {          // A block (i, j), i <= j, and its mirror
            const int i = tri[2 * it], j = tri[2 * it + 1];
            const int ai = pr[2 * i], bi = pr[2 * i + 1], aj = pr[2 * j], bj = pr[2 * j + 1];
            double ci, si, cj, sj;
            rot(Ao, ai, bi, ci, si);
            if (i == j) cj = ci, sj = si;
            else rot(Ao, aj, bj, cj, sj);
            const double x00 = Ao[ai * LDS + aj], x01 = Ao[ai * LDS + bj];
            const double x10 = Ao[bi * LDS + aj], x11 = Ao[bi * LDS + bj];
            // J_i^T X
            const double y00 = ci * x00 - si * x10, y01 = ci * x01 - si * x11;
            const double y10 = si * x00 + ci * x10, y11 = si * x01 + ci * x11;
            // (J_i^T X) J_j
            const double z00 = y00 * cj - y01 * sj, z01 = y00 * sj + y01 * cj;
            const double z10 = y10 * cj - y11 * sj, z11 = y10 * sj + y11 * cj;
            An[ai * LDS + aj] = z00;
            An[ai * LDS + bj] = z01;
            An[bi * LDS + aj] = z10;
            An[bi * LDS + bj] = z11;
            if (i != j) {
              An[aj * LDS + ai] = z00;
              An[bj * LDS + ai] = z01;
              An[aj * LDS + bi] = z10;
              An[bj * LDS + bi] = z11;
            }
          } else {                  // V block: rows of pair i, columns of pair j
            const int r = it - ntri, i = r / half, j = r % half;
            const int ai = pr[2 * i], bi = pr[2 * i + 1], aj = pr[2 * j], bj = pr[2 * j + 1];
            double cj, sj;
            rot(Ao, aj, bj, cj, sj);
            if (sj == 0.0) continue;
            const double v00 = V[ai * LDS + aj], v01 = V[ai * LDS + bj];
            const double v10 = V[bi * LDS + aj], v11 = V[bi * LDS + bj];
            V[ai * LDS + aj] = v00 * cj - v01 * sj;
            V[ai * LDS + bj] = v00 * sj + v01 * cj;
            V[bi * LDS + aj] = v10 * cj - v11 * sj;
            V[bi * LDS + bj] = v10 * sj + v11 * cj;
          }
        }
        cur ^= 1;
        __syncthreads();
  #ifdef SBT_RITZ_CLOCK
        if (tid == 0) g_ritz_clock[15] += clock64() - c0;
  #endif
      }
    }
    const double* A = smr + cur * MAT;
    t_jacobi = clock64();
    RITZ_STAMP(5);

    // descending order of the p true eigenvalues (the padding index is excluded)
    if (tid < p) {
      const double d = A[tid * LDS + tid];
      int pos = 0;
      for (int j = 0; j < p; ++j) {
        const double dj = A[j * LDS + j];
        pos += (dj > d) || (dj == d && j < tid);
      }
      perm[pos] = tid;
    }
    if (tid < kMaxP) {
      res[tid] = 0.0;
      amax[tid] = 0.0;
      s_arg[tid] = 0x7fffffff;
    }
    __syncthreads();
    for (int e = tid; e < p * rank; e += kThreads) {
      const int l = e / rank, j = e % rank;
      Vs[l * LDS + j] = V[l * LDS + perm[j]];
    }
    if (tid < rank) {
      wv[tid] = A[perm[tid] * LDS + perm[tid]];
      w[tid] = wv[tid];
    }
  }
  RITZ_STAMP(6);
  // ---- Ritz vectors, residuals and sign rule on all CTAs of the cluster ----
  cluster.sync();
  RITZ_STAMP(7);
  if (crank != 0) {  // copy the sorted eigenvectors / values from CTA 0
    const double* rVs = cluster.map_shared_rank(Vs, 0);
    const double* rwv = cluster.map_shared_rank(wv, 0);
    for (int e = tid; e < p * rank; e += kThreads) {
      const int l = e / rank, j = e % rank;
      Vs[l * LDS + j] = rVs[l * LDS + j];
    }
    if (tid < rank) wv[tid] = rwv[tid];
  }
  if (tid < kMaxP) {
    res[tid] = 0.0;
    amax[tid] = 0.0;
    s_arg[tid] = 0x7fffffff;
  }
  __syncthreads();  // A / V are dead from here: region 0 holds Q / Z tiles
  const double wmax = fmax(wv[0], 0.0);

  // U = Q V_r, Y = Z V_r over row tiles (tile t on CTA t % kCluster);
  // thread = (row r, 8-column group g)
  const int r = tid % kTileRows, g = tid / kTileRows;  // 8 groups of 8 columns
  const int ngroups = (rank + 7) / 8;
  double rsum[8], mx[8];
  int ax[8];
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) rsum[jj] = 0.0, mx[jj] = -1.0, ax[jj] = 0x7fffffff;
  for (int64_t i0 = int64_t(crank) * kTileRows; i0 < n; i0 += kCluster * kTileRows) {
    const int rows = n - i0 < kTileRows ? int(n - i0) : kTileRows;
    load_tile(i0, rows);
    __syncthreads();
    {  // U_t = Q_t V_r, Y_t = Z_t V_r on the fp64 tensor pipe -> Us / Yv
      const int warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fk = lane & 3;
      const int ntj = (rank + 7) >> 3;
      for (int t = warp; t < 2 * 8 * ntj; t += kThreads / 32) {
        const int which = t / (8 * ntj), rem = t % (8 * ntj), mt = rem / ntj, nj = rem % ntj;
        const double* src = which ? Zs : Qs;
        const int i = 8 * mt + fr, j = 8 * nj + fr;
        double c[8][2];     // k-step s -> chain s % 8 (independent DMMAs)
#pragma unroll
        for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
        for (int l0 = 0; l0 < p; l0 += 32) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int l = l0 + 4 * q + fk;
            dmma(c[q], l < p ? src[l * LDT + i] : 0.0, l < p ? Vs[l * LDS + j] : 0.0);
          }
        }
        double* dst = which ? Yv : Us;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 8 * nj + 2 * fk + h;
          double v = 0.0;
#pragma unroll
          for (int q = 0; q < 8; ++q) v += c[q][h];
          if (col < rank) dst[i * LDS + col] = v;
        }
      }
    }
    __syncthreads();
    if (g < ngroups) {
      const int j0 = 8 * g;
      double u[8], y[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        u[jj] = j0 + jj < rank ? Us[r * LDS + j0 + jj] : 0.0;
        y[jj] = j0 + jj < rank ? Yv[r * LDS + j0 + jj] : 0.0;
      }
      if (r < rows) {
        const int64_t i = i0 + r;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          if (j0 + jj >= rank) break;
          const double d = y[jj] - wv[j0 + jj] * u[jj];
          rsum[jj] = fma(d, d, rsum[jj]);
          const double au = fabs(u[jj]);
          if (au > mx[jj]) mx[jj] = au, ax[jj] = int(i);  // i ascending
          ut[int64_t(j0 + jj) * n + i] = u[jj];
          if (yt) yt[int64_t(j0 + jj) * n + i] = y[jj];
        }
      }
    }
    __syncthreads();  // the tile buffers are reused
  }
  // per-CTA column reductions: residual sums, then (max |u|, first index)
  if (g < ngroups) {  // warp-uniform (a warp shares g)
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int j = 8 * g + jj;
      if (j >= rank) break;
      double rr = rsum[jj], a = mx[jj];
      int x = ax[jj];
      for (int o = 16; o > 0; o >>= 1) {
        rr += __shfl_xor_sync(0xffffffffu, rr, o);
        const double ao = __shfl_xor_sync(0xffffffffu, a, o);
        const int xo = __shfl_xor_sync(0xffffffffu, x, o);
        if (ao > a || (ao == a && xo < x)) a = ao, x = xo;
      }
      if ((tid & 31) == 0) {
        atomicAdd(&res[j], rr);
        // max first (a >= 0: bit order == value order), then the smallest
        // index attaining it
        if (a >= 0.0)
          atomicMax(reinterpret_cast<unsigned long long*>(&amax[j]), __double_as_longlong(a));
      }
      mx[jj] = a;
      ax[jj] = x;
    }
  }
  __syncthreads();
  if (g < ngroups) {
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int j = 8 * g + jj;
      if (j >= rank) break;
      if ((tid & 31) == 0 && mx[jj] == amax[j]) atomicMin(&s_arg[j], ax[jj]);
    }
  }
  RITZ_STAMP(8);
  __threadfence();  // U entries (global) visible to the cluster after the barrier
  cluster.sync();
  const long long t_ritz = clock64();
  RITZ_STAMP(9);
  // sign rule (tucker.py:71-75): combine the CTAs' (max, first index) per
  // column, then every CTA negates its own rows of negative columns
  if (tid < rank) {
    double best = -1.0;
    int arg = 0x7fffffff;
#pragma unroll
    for (int c = 0; c < kCluster; ++c) {
      const double a = *cluster.map_shared_rank(amax + tid, c);
      const int x = *cluster.map_shared_rank(s_arg + tid, c);
      if (a > best || (a == best && x < arg)) best = a, arg = x;
    }
    sgn[tid] = ut[int64_t(tid) * n + arg] < 0.0 ? -1.0 : 1.0;
  }
  cluster.sync();  // every CTA has read its reference entries before any negation
  for (int64_t i0 = int64_t(crank) * kTileRows; i0 < n; i0 += kCluster * kTileRows) {
    const int rows = n - i0 < kTileRows ? int(n - i0) : kTileRows;
    for (int e = tid; e < rank * kTileRows; e += kThreads) {
      const int j = e / kTileRows, rr = e % kTileRows;
      if (rr >= rows) continue;
      double* u = ut + int64_t(j) * n + i0 + rr;
      if (sgn[j] < 0.0) *u = -*u;
      if (ut32) ut32[int64_t(j) * n + i0 + rr] = float(*u);
    }
  }
  if (crank == 0 && tid < 32) {  // one warp: residual norms and the flag
    double rmax = 0.0;
    for (int j = tid; j < rank; j += 32) {
      double rj = 0.0;
#pragma unroll
      for (int c = 0; c < kCluster; ++c) rj += *cluster.map_shared_rank(res + j, c);
      rmax = fmax(rmax, sqrt(rj));
    }
    for (int o = 16; o > 0; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    if (tid == 0) {
      const bool ok = wmax > 0.0 && rmax <= tol * wmax;
      flag[0] = ok ? 1 : 0;
      rel[0] = wmax > 0.0 ? rmax / wmax : 0.0;
      rel[1] = double(sweeps);
      rel[2] = double(t_jacobi - t_start);  // diagnostics: SM cycles per phase
      rel[3] = double(t_ritz - t_jacobi);
      rel[4] = double(clock64() - t_ritz);
      rel[5] = double(newton);
    }
  }
  RITZ_STAMP(10);
  cluster.sync();  // no CTA exits while its shared memory may still be read
  RITZ_STAMP(11);
}

}  // namespace ritz
}  // namespace sbt
