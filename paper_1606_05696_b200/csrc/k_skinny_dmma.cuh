// Skinny fp64 GEMMs (N <= 64 after orientation): the HOOI factor
// update's rank-p products (Y^T Q: 1024 x 32 x 512, Y W: 512 x 32 x 1024,
// [Q Z]^T Z: 64 x 32 x 512).  The 128 x 128 DMMA tiles of k_dmma.cuh waste 3/4
// of every tile on a 32-wide N and leave most SMs idle; here a CTA computes a
// 64 x 32 tile over one K-split (4 warps, each 16 x 32 = 2 x 4 DMMA m8n8k4
// fragments), enough splits to fill the GPU, and the partial tiles are summed
// in a fixed split order by the last CTA of each tile (an atomic ticket per
// tile), so the result is deterministic and there is no second kernel.
// Batched calls (fp64 Tucker mode products, N = rank) run one grid z-slice per
// batch entry without splitting K.
#pragma once
#include "sbt_common.cuh"

namespace sbt {
namespace skinny {

constexpr int BM = 64, BN = 32, KC = 64, NT = 128;
constexpr int LDK = KC + 4;  // [mn][k] rows (K-major operands)
constexpr int LDMA = BM + 4; // [k][m]   (MN-major A)
constexpr int LDNB = BN + 4; // [k][n]   (N-major B)
constexpr int A_DOUBLES = BM * LDK > KC * LDMA ? BM * LDK : KC * LDMA;
constexpr int B_DOUBLES = BN * LDK > KC * LDNB ? BN * LDK : KC * LDNB;
constexpr int SMEM_BYTES = 2 * (A_DOUBLES + B_DOUBLES) * 8;  // double-buffered
constexpr int TILE = BM * BN;

// 8-byte async copy global -> shared, zero-filled when !valid
__device__ __forceinline__ void cp8(double* smem, const double* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem),
               "r"(valid ? 8 : 0)
               : "memory");
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// A_K: A[m][k] with k unit-stride (else m unit-stride); B_K: B[k][n] with k
// unit-stride (else n unit-stride).  grid = (tiles, splits); ws / cnt are
// needed when splits > 1 (cnt zeroed by the caller).
template <bool A_K, bool B_K>
__global__ void __launch_bounds__(NT) skinny_dmma_kernel(GemmParams<double> p, int tiles_m,
                                                         int64_t kper, double* __restrict__ ws,
                                                         unsigned* __restrict__ cnt) {
  extern __shared__ __align__(16) double smk[];
  double* sa = smk;
  double* sb = smk + 2 * A_DOUBLES;  // [2][B_DOUBLES] after the two A buffers
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int tile = blockIdx.x, split = blockIdx.y, S = gridDim.y;
  const int64_t m0 = int64_t(tile % tiles_m) * BM, n0 = int64_t(tile / tiles_m) * BN;
  const int64_t kb = int64_t(split) * kper;
  const int64_t ke = kb + kper < p.k ? kb + kper : p.k;
  // batched calls (no split): blockIdx.z = batch entry (batch2 outer)
  const int64_t zb = blockIdx.z % p.batch, zq = blockIdx.z / p.batch;
  const double* __restrict__ A = p.a + zb * p.aps + zq * p.aps2;
  const double* __restrict__ B = p.b + zb * p.bps + zq * p.bps2;
  double* __restrict__ Cz = p.c + zb * p.cps + zq * p.cps2;

  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // K-chunks of KC through a two-buffer cp.async ring: chunk c + 1 is in
  // flight while chunk c is multiplied
  auto stage = [&](int64_t k0, int buf) {
    double* as = sa + buf * A_DOUBLES;
    double* bs = sb + buf * B_DOUBLES;
    const int kn = ke - k0 < KC ? int(ke - k0) : KC;
    if (A_K) {
      for (int e = tid; e < BM * KC; e += NT) {
        const int m = e / KC, k = e % KC;
        const bool in = m0 + m < p.m && k < kn;
        cp8(as + m * LDK + k, in ? A + (m0 + m) * p.ars + k0 + k : A, in);
      }
    } else {
      for (int e = tid; e < BM * KC; e += NT) {
        const int m = e % BM, k = e / BM;
        const bool in = m0 + m < p.m && k < kn;
        cp8(as + k * LDMA + m, in ? A + (m0 + m) + (k0 + k) * p.acs : A, in);
      }
    }
    if (B_K) {
      for (int e = tid; e < BN * KC; e += NT) {
        const int n = e / KC, k = e % KC;
        const bool in = n0 + n < p.n && k < kn;
        cp8(bs + n * LDK + k, in ? B + (k0 + k) + (n0 + n) * p.bcs : B, in);
      }
    } else {
      for (int e = tid; e < BN * KC; e += NT) {
        const int n = e % BN, k = e / BN;
        const bool in = n0 + n < p.n && k < kn;
        cp8(bs + k * LDNB + n, in ? B + (k0 + k) * p.brs + n0 + n : B, in);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int nch = ke > kb ? int((ke - kb + KC - 1) / KC) : 0;
  if (nch > 0) stage(kb, 0);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      stage(kb + int64_t(c + 1) * KC, (c + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* as = sa + (c & 1) * A_DOUBLES;
    const double* bs = sb + (c & 1) * B_DOUBLES;
    const int64_t k0 = kb + int64_t(c) * KC;
    const int kn = ke - k0 < KC ? int(ke - k0) : KC;
    const int kq = (kn + 3) & ~3;
    for (int kk = 0; kk < kq; kk += 4) {
      double af[2], bf[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int m = warp * 16 + i * 8 + fr;
        af[i] = A_K ? as[m * LDK + kk + fk] : as[(kk + fk) * LDMA + m];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = j * 8 + fr;
        bf[j] = B_K ? bs[n * LDK + kk + fk] : bs[(kk + fk) * LDNB + n];
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
    __syncthreads();
  }

  if (S == 1) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int64_t row = m0 + warp * 16 + i * 8 + fr;
      if (row >= p.m) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t col = n0 + j * 8 + 2 * fk + h;
          if (col < p.n) store_out(Cz + row * p.crs + col * p.ccs, acc[i][j][h], p.alpha, p.beta);
        }
    }
    return;
  }
  // split-K: partial tile -> workspace; the last CTA of the tile reduces
  double* part = ws + (int64_t(tile) * S + split) * TILE;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        part[(warp * 16 + i * 8 + fr) * BN + j * 8 + 2 * fk + h] = acc[i][j][h];
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&cnt[tile], 1u) == unsigned(S - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // fixed split order; the partial loads of 4 element pairs x 8 splits are in
  // flight together (the reduction is latency-bound, not bandwidth-bound)
  const double2* tp = reinterpret_cast<const double2*>(ws + int64_t(tile) * S * TILE);
  constexpr int PAIRS = TILE / 2 / NT;  // 8 element pairs per thread
#pragma unroll 1
  for (int q0 = 0; q0 < PAIRS; q0 += 4) {
    double2 sum[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) sum[q] = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int s0 = 0; s0 < S; s0 += 8) {
      double2 v[8][4];
#pragma unroll
      for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          v[s][q] = s0 + s < S ? __ldcg(tp + int64_t(s0 + s) * (TILE / 2) + tid + (q0 + q) * NT)
                               : make_double2(0.0, 0.0);
#pragma unroll
      for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (s0 + s < S) {
            sum[q].x += v[s][q].x;
            sum[q].y += v[s][q].y;
          }
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = 2 * (tid + (q0 + q) * NT);
      const int64_t row = m0 + e / BN, col = n0 + e % BN;
      if (row >= p.m) continue;
      if (col < p.n) store_out(Cz + row * p.crs + col * p.ccs, sum[q].x, p.alpha, p.beta);
      if (col + 1 < p.n) store_out(Cz + row * p.crs + (col + 1) * p.ccs, sum[q].y, p.alpha, p.beta);
    }
  }
}

}  // namespace skinny
}  // namespace sbt
