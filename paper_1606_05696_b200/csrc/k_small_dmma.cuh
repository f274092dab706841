// K3 (fp64, 16 < n <= 64): small-matrix batched GEMM on the DMMA pipe.
//
// The SIMT K3 kernel (k_small.cuh) reaches 0.93-0.95 of HBM bandwidth for fp64
// n <= 16, but at n = 32 (AI = 2.7 flop/B) it is shared-memory bound: a 4x4
// register block reads 4 bytes of shared memory per DFMA.  Here each warp owns
// one matrix and runs the whole 32x32x32 product as 128 DMMA.8x8x4 with every
// fragment loaded once per k-step (0.5 B of shared memory per FMA).
//
// Operand staging: one 3-D TMA box per operand per group of G matrices,
// (rows, cols, G) with the row extent padded to LD = rows + 4 doubles.  The
// TMA zero-fills the out-of-range rows, so the box lands as [matrix][col][LD]
// with a column stride of LD (== 4 mod 16 doubles): the DMMA fragment loads
// (8 rows x 4 columns per half-warp) hit 16 distinct bank pairs -- no
// conflicts, no padding copy.
//
// The product is computed transposed, C^T = B^T A^T (MMA M = C column j, MMA
// N = C row i), so each thread's accumulator pair is two consecutive rows of a
// column of C: one 16-byte store.
//
// NMAX = 64 (32 < n <= 64, AI 5.3 flop/B: compute-bound in fp64): four warps
// share one matrix, each owning a 32 x 32 quadrant of C^T; one matrix per
// stage (70 KB), three stages.
//
// Requires A stored with rows contiguous (ars = 1, acs = m), B with k
// contiguous (brs = 1, bcs = k), C dense (crs = 1, ccs = m); m, n multiples of
// 8 and <= NMAX, k a multiple of 4 and <= NMAX (checked by the dispatcher).
#pragma once
#include <cuda.h>

#include "sbt_common.cuh"
#include "sm100_ptx.cuh"

namespace sbt {
namespace small_dmma {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;

__host__ __device__ constexpr int ld_of(int rows) { return ((rows + 15) / 16) * 16 + 4; }
template <int NMAX>
struct Cfg {
  static constexpr int Q = NMAX / 32;            // quadrants per side
  static constexpr int WPM = Q * Q;              // warps per matrix
  static constexpr int G = kWarps / WPM;         // matrices per group
  static constexpr int LD_MAX = NMAX + 4;        // padded leading dimension
  static constexpr int STAGE_DOUBLES = G * 2 * LD_MAX * NMAX;
  // three one-stage CTAs per SM (12 warps) instead of one three-stage CTA
  // (4 warps): the DMMA pipe needs more than one warp per scheduler, and while
  // one CTA waits for its next group the others compute.  Measured at P = 10^6
  // (n = 32) / 2 x 10^5 (n = 64): 0.84 -> 1.02 of the copy-measured HBM rate,
  // 17.5 -> 24.9 TFLOP/s
#ifndef SBT_SMALL_DMMA64_CTAS
#define SBT_SMALL_DMMA64_CTAS 3
#endif
#ifndef SBT_SMALL_DMMA32_CTAS
#define SBT_SMALL_DMMA32_CTAS 3
#endif
  static constexpr int CTAS_PER_SM = NMAX == 64 ? SBT_SMALL_DMMA64_CTAS : SBT_SMALL_DMMA32_CTAS;
  static constexpr int STAGES = CTAS_PER_SM >= 3 ? 1 : 3 / CTAS_PER_SM;
  static constexpr int SMEM_BYTES = STAGES * STAGE_DOUBLES * 8 + 64;
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(ptx::smem_addr(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(ptx::smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

template <int NMAX>
__global__ void __launch_bounds__(kThreads, Cfg<NMAX>::CTAS_PER_SM)
small_dmma_kernel(GemmParams<double> p, const __grid_constant__ CUtensorMap tmA,
                  const __grid_constant__ CUtensorMap tmB, int64_t ngroups) {
  using C_ = Cfg<NMAX>;
  constexpr int G = C_::G, STAGES = C_::STAGES;
  auto stage_doubles = [] { return C_::STAGE_DOUBLES; };
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + STAGES * stage_doubles() * 8);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = int(p.m), n = int(p.n), k = int(p.k);
  const int lda = ld_of(m), ldb = ld_of(k);
  const int a_doubles = lda * k, b_doubles = ldb * n;  // one matrix, padded
  const uint32_t tx = uint32_t(G * (a_doubles + b_doubles) * 8);

  auto issue = [&](int64_t grp, int slot) {
    double* sa = sm + slot * stage_doubles();
    double* sb = sa + G * a_doubles;
    ptx::mbar_arrive_expect_tx(&full[slot], tx);
    tma_load_3d(sa, &tmA, &full[slot], 0, 0, int(grp * G));
    tma_load_3d(sb, &tmB, &full[slot], 0, 0, int(grp * G));
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) ptx::mbar_init(&full[s], 1);
    ptx::fence_mbarrier_init();
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      const int64_t gi = blockIdx.x + int64_t(s) * gridDim.x;
      if (gi < ngroups) issue(gi, s);
    }
  }
  __syncthreads();

  const int mt = m >> 3, nt = n >> 3;      // C row / column tiles of 8
  const int r4 = lane & 3, q8 = lane >> 2;  // fragment coordinates
  const bool vec = p.beta == 0.0 && (p.ccs % 2 == 0) && (p.cps % 2 == 0) &&
                   ((reinterpret_cast<uintptr_t>(p.c) & 15) == 0);
  uint32_t it = 0;
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++it) {
    const int slot = int(it % STAGES);
    ptx::mbar_wait(&full[slot], (it / STAGES) & 1u);
    const int mat = warp / C_::WPM, qw = warp % C_::WPM;
    const int jq = qw / C_::Q, iq = qw % C_::Q;  // this warp's quadrant of C^T
    const int64_t bidx = grp * G + mat;
    if (bidx < p.batch) {
      const double* sa = sm + slot * stage_doubles() + mat * a_doubles + 32 * iq;
      const double* sb = sm + slot * stage_doubles() + G * a_doubles + mat * b_doubles +
                         32 * jq * ldb;
      const int nt_q = nt - 4 * jq, mt_q = mt - 4 * iq;  // tiles in this quadrant
      double acc[4][4][2];  // [j tile][i tile][pair]
#pragma unroll
      for (int jt = 0; jt < 4; ++jt)
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) acc[jt][i2][0] = acc[jt][i2][1] = 0.0;
      for (int l0 = 0; l0 < k; l0 += 4) {
        double fa[4], fb[4];
        // MMA A = B^T (8 j x 4 l): thread (j = q8, l = r4) -> B[l + j*ldb]
        // MMA B = A^T (4 l x 8 i): thread (l = r4, i = q8) -> A[i + l*lda]
#pragma unroll
        for (int jt = 0; jt < 4; ++jt)
          fa[jt] = jt < nt_q ? sb[(l0 + r4) + (8 * jt + q8) * ldb] : 0.0;
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2)
          fb[i2] = i2 < mt_q ? sa[(8 * i2 + q8) + (l0 + r4) * lda] : 0.0;
#pragma unroll
        for (int jt = 0; jt < 4; ++jt)
#pragma unroll
          for (int i2 = 0; i2 < 4; ++i2)
            if (jt < nt_q && i2 < mt_q) dmma(acc[jt][i2], fa[jt], fb[i2]);
      }
      // D[j][i] (j = 8 jt + q8, i = 8 i2 + 2 r4 + {0,1}) = C[i + j*ccs]
      double* C = p.c + bidx * p.cps + 32 * iq + int64_t(32 * jq) * p.ccs;
#pragma unroll
      for (int jt = 0; jt < 4; ++jt) {
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) {
          if (jt >= nt_q || i2 >= mt_q) continue;
          double* dst = C + (8 * i2 + 2 * r4) + int64_t(8 * jt + q8) * p.ccs;
          if (vec) {
            *reinterpret_cast<double2*>(dst) =
                make_double2(p.alpha * acc[jt][i2][0], p.alpha * acc[jt][i2][1]);
          } else {
            store_out(dst, acc[jt][i2][0], p.alpha, p.beta);
            store_out(dst + 1, acc[jt][i2][1], p.alpha, p.beta);
          }
        }
      }
    }
    __syncthreads();  // every warp is done with this slot
    const int64_t gnext = grp + int64_t(STAGES) * gridDim.x;
    if (tid == 0 && gnext < ngroups) issue(gnext, slot);
  }
}

}  // namespace small_dmma
}  // namespace sbt
