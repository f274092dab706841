// K1 (fp64): strided batched GEMM on the fp64 tensor pipe (DMMA).
//
// tcgen05.mma has no f64 kind (ptxas rejects .kind::f64), so the B200 fp64
// tensor path is the warp-level mma.sync m8n8k4 f64, which is the native
// DMMA.8x8x4 SASS instruction.  Every DMMA is an IEEE fp64 fused multiply-add
// chain per output element, so results agree with the fp64 CPU oracle to a
// few ulp (reference tolerance 1e-12, test_acceptance.py:79).
//
// Staging: 3-stage cp.async (16 B) ring into padded shared-memory tiles whose
// contiguous mode is the operand's unit-stride global mode (K-major -> [mn][k],
// MN-major -> [k][mn]); the paddings (20 / 132 doubles) make every fragment
// load bank-conflict free.  Out-of-range chunks are zero-filled.
//
// CTA tile 128 x 128 x 16, 8 warps as 2 (M) x 4 (N), warp tile 64 x 32 =
// 8 x 4 DMMA tiles (64 fp64 accumulators per thread).
#pragma once
#include "sbt_common.cuh"

namespace sbt {
namespace dmma {

#ifndef SBT_DMMA_BK
#define SBT_DMMA_BK 16
#endif
#ifndef SBT_DMMA_STAGES
#define SBT_DMMA_STAGES 3
#endif
constexpr int BM = 128, BN = 128, BK = SBT_DMMA_BK, STAGES = SBT_DMMA_STAGES;
static_assert(BK == 16 || BK == 32, "K-block depth");
constexpr int kThreads = 256;      // staging loops assume >= 256 threads
template <int NW>
struct WarpGrid {                    // NW = 8: 2 x 4 warps of 64 x 32; 16: 4 x 4 of 32 x 32
  static constexpr int WM = NW / 4, TM = 128 / WM / 8;  // warp rows, DMMA tiles per warp row
};
constexpr int LDK = BK + 4;   // [mn][k] rows (BK k + 4 pad: rows 8 words apart in the banks)
constexpr int LDMN = 132; // [k][mn] rows (128 mn + 4 pad)
// Batch-blocked A (the exceptional cases: A unit-stride along the batch, B
// batch-independent): the tile's 128 MMA rows are 4 batch entries x 32 m,
// MMA row R = 32 b + m.  A is staged with 8-byte cp.async, lanes walking the
// batch fastest (coalesced: 4 entries = one 32 B sector), into [k][LDBB] rows
// with smem position 36 b + m -- 2 wavefronts per warp store (the minimum for
// 8 B x 32 lanes) and, with LDBB = 148 = 4 mod 16, conflict-free fragment
// loads.  A fragment (8 consecutive R) is 8 consecutive m of one batch entry,
// so the epilogue stores 64-byte runs of C exactly as for plain tiles.
constexpr int LDBB = 148;
constexpr int TILE_RAW = 128 * LDK > BK * LDMN ? 128 * LDK : BK * LDMN;  // BK 16: 2560 vs 2112
constexpr int TILE_DOUBLES = TILE_RAW > BK * LDBB ? TILE_RAW : BK * LDBB;
constexpr int SMEM_BYTES = STAGES * 2 * TILE_DOUBLES * 8;                   // 120 KB
// BNT = 64 tiles: the B half is 64 x BK (K-major) or BK x LDMN (MN-major)
constexpr int B64_DOUBLES = 64 * LDK > BK * LDMN ? 64 * LDK : BK * LDMN;
constexpr int SMEM_BYTES_N64 = STAGES * (TILE_DOUBLES + B64_DOUBLES) * 8;   // 109.5 KB at BK 16

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// Stage one operand tile (rows = MN extent 128, k = 16) with 16-byte cp.async.
// KMAJ: global k unit-stride -> smem [mn][LDK]; else mn unit-stride -> [k][LDMN].
template <bool KMAJ, int NT = kThreads, int ROWS = 128>
__device__ __forceinline__ void stage_operand(double* dst, const double* __restrict__ src,
                                              int64_t mn0, int64_t k0, int64_t mn_ext,
                                              int64_t k_ext, int64_t s_mn, int64_t s_k, int tid) {
#pragma unroll
  for (int i = 0; i < ROWS * BK / 2 / NT; ++i) {  // ROWS x BK doubles in 16-byte chunks
    const int e = tid + i * NT;
    if (KMAJ) {
      const int mn = e / (BK / 2), k2 = (e % (BK / 2)) * 2;
      const int64_t gm = mn0 + mn, gk = k0 + k2;
      const bool ok = gm < mn_ext && gk < k_ext;
      cp_async16(dst + mn * LDK + k2, ok ? src + gm * s_mn + gk : src, ok);
    } else {
      const int k = e / (ROWS / 2), mn2 = (e % (ROWS / 2)) * 2;
      const int64_t gm = mn0 + mn2, gk = k0 + k;
      const bool ok = gm < mn_ext && gk < k_ext;
      cp_async16(dst + k * LDMN + mn2, ok ? src + gm + gk * s_k : src, ok);
    }
  }
}

// BB A staging: 128 rows (4 batch x 32 m) x BK k, 8-byte chunks
template <int NT = kThreads>
__device__ __forceinline__ void stage_bb(double* dst, const double* __restrict__ src, int64_t b0,
                                         int64_t m0, int64_t k0, int64_t nbatch, int64_t m_ext,
                                         int64_t k_ext, int64_t ars, int64_t acs, int tid) {
#pragma unroll
  for (int i = 0; i < 128 * BK / NT; ++i) {
    const int e = tid + i * NT;
    const int k = e >> 7, b = e & 3, m = (e >> 2) & 31;
    const int64_t gb = b0 + b, gm = m0 + m, gk = k0 + k;
    const bool ok = gb < nbatch && gm < m_ext && gk < k_ext;
    cp_async8(dst + k * LDBB + 36 * b + m, ok ? src + gb + gm * ars + gk * acs : src, ok);
  }
}

// BNT: N extent of the CTA tile.  128 (one CTA per SM; NW = 8 or 16); 64
// with NW = 8 (4 x 2 warps of 32 x 32, <= 128 registers) runs two CTAs per
// SM, so one CTA's prologue / epilogue overlaps the other's main loop.
// BB A staging with 16-byte copies: the two batch entries (b, b+1) of a pair
// are adjacent in global memory (the batch is A's unit-stride mode), so they
// land side by side: position k * LDB2 + (b >> 1) * 64 + 2 m + (b & 1).
// Half the copy instructions of stage_bb; needs ars, acs even and A 16-byte
// aligned (checked by the launcher).
constexpr int LDB2 = 132;
static_assert(BK * LDB2 <= TILE_DOUBLES, "BB16 tile fits the stage");
template <int NT = kThreads>
__device__ __forceinline__ void stage_bb16(double* dst, const double* __restrict__ src,
                                           int64_t b0, int64_t m0, int64_t k0, int64_t nbatch,
                                           int64_t m_ext, int64_t k_ext, int64_t ars,
                                           int64_t acs, int tid) {
#pragma unroll
  for (int i = 0; i < 64 * BK / NT; ++i) {
    const int e = tid + i * NT;
    const int k = e >> 6, pr = e & 1, m = (e >> 1) & 31;
    const int64_t gb = b0 + 2 * pr, gm = m0 + m, gk = k0 + k;
    double* d = dst + k * LDB2 + pr * 64 + 2 * m;
    const bool row = gm < m_ext && gk < k_ext;
    const double* s = src + gb + gm * ars + gk * acs;
    if (row && gb + 1 < nbatch) {
      cp_async16(d, s, true);
    } else {                         // batch tail: one entry or none
      cp_async8(d, row && gb < nbatch ? s : src, row && gb < nbatch);
      cp_async8(d + 1, src, false);
    }
  }
}

template <bool A_K, bool B_K, bool BB = false, int NW = 8, int BNT = 128, bool BB16 = false>
__global__ void __launch_bounds__(NW * 32, BNT <= 64 ? 2 : 1)
dmma_gemm_kernel(GemmParams<double> p, int64_t tiles_m, int64_t tiles_n) {
  extern __shared__ __align__(16) double sm[];
  static_assert(BNT == 128 || (BNT <= 64 && NW == 8), "tile configurations");
  constexpr int NT = NW * 32;
  constexpr int WN = BNT / 32;                       // warps along N (32 columns each)
  constexpr int WM = NW / WN, TM = 128 / WM / 8;     // warps along M, DMMA row tiles per warp
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp % WM, wn = warp / WM;  // WM x 4 warps

  int64_t t = blockIdx.x;
  const int64_t m0 = (t % tiles_m) * (BB ? 32 : BM);
  t /= tiles_m;
  const int64_t n0 = (t % tiles_n) * BNT;
  t /= tiles_n;
  const int64_t nbatch = BB ? (p.batch + 3) / 4 : p.batch;
  const int64_t pb = t % nbatch, qb = t / nbatch;
  const double* __restrict__ A = p.a + (BB ? 0 : pb * p.aps) + qb * p.aps2;
  const double* __restrict__ B = p.b + (BB ? 0 : pb * p.bps) + qb * p.bps2;
  const int nkb = int((p.k + BK - 1) / BK);

  constexpr int STAGE_D = TILE_DOUBLES + (BNT == 128 ? TILE_DOUBLES : B64_DOUBLES);
  auto stage = [&](int kb) {
    double* sa = sm + (kb % STAGES) * STAGE_D;
    double* sb = sa + TILE_DOUBLES;
    const int64_t k0 = int64_t(kb) * BK;
    if (BB && BB16)
      stage_bb16<NT>(sa, A, pb * 4, m0, k0, p.batch, p.m, p.k, p.ars, p.acs, tid);
    else if (BB)
      stage_bb<NT>(sa, A, pb * 4, m0, k0, p.batch, p.m, p.k, p.ars, p.acs, tid);
    else
      stage_operand<A_K, NT>(sa, A, m0, k0, p.m, p.k, A_K ? p.ars : 1, A_K ? 1 : p.acs, tid);
    stage_operand<B_K, NT, BNT>(sb, B, n0, k0, p.n, p.k, B_K ? p.bcs : 1, B_K ? 1 : p.brs, tid);
  };

  double acc[TM][4][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkb) stage(s);
    cp_async_commit();
  }
  const int fr = lane >> 2, fk = lane & 3;  // fragment row (mn) / k within a DMMA
  for (int kb = 0; kb < nkb; ++kb) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (kb + STAGES - 1 < nkb) stage(kb + STAGES - 1);
    cp_async_commit();
    const double* sa = sm + (kb % STAGES) * STAGE_D;
    const double* sb = sa + TILE_DOUBLES;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[TM], bf[4];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int m = wm * (TM * 8) + i * 8 + fr;
        if (BB && BB16)
          af[i] = sa[(kk + fk) * LDB2 + ((m >> 5) >> 1) * 64 + 2 * (m & 31) + ((m >> 5) & 1)];
        else if (BB) af[i] = sa[(kk + fk) * LDBB + 36 * (m >> 5) + (m & 31)];
        else af[i] = A_K ? sa[m * LDK + kk + fk] : sa[(kk + fk) * LDMN + m];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = wn * 32 + j * 8 + fr;
        bf[j] = B_K ? sb[n * LDK + kk + fk] : sb[(kk + fk) * LDMN + n];
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  double* C = p.c + (BB ? 0 : pb * p.cps) + qb * p.cps2;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int R = wm * (TM * 8) + i * 8 + fr;
    const int64_t row = BB ? m0 + (R & 31) : m0 + R;
    if (row >= p.m) continue;
    if (BB && pb * 4 + (R >> 5) >= p.batch) continue;
    double* Cr = BB ? C + (pb * 4 + (R >> 5)) * p.cps : C;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t col = n0 + wn * 32 + j * 8 + 2 * fk + h;
        if (col < p.n) store_out(Cr + row * p.crs + col * p.ccs, acc[i][j][h], p.alpha, p.beta);
      }
    }
  }
}

}  // namespace dmma
}  // namespace sbt
