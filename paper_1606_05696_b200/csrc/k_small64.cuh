// K3 (fp32, n = 64): batched 64 x 64 x 64 products with 8 x 8 register blocks.
//
// At n = 64 the fp32 batched product needs 70 TFLOP/s to keep up with HBM
// (AI = 10.7 flop/B).  The generic K3 kernel's 4 x 4 blocks read 0.5 float of
// shared memory per FMA, which caps it at half the FFMA rate; here each thread
// owns an 8 x 8 block (16 shared-memory floats per 64 FMAs), so shared-memory
// bandwidth matches the FFMA rate.
//
// Staging: one 3-D TMA box per operand per group of G matrices; B's column
// stride is padded to 68 floats by TMA zero fill.  A thread owns rows
// i0..i0+7 and the strided columns j0, j0+8, ..., j0+56: the eight j0 lanes of
// a quarter-warp then read columns 68 floats apart -- distinct banks -- and the
// A reads are broadcasts of one 256-byte column run.
//
// Requires A stored with rows contiguous (ars = 1, acs = m), B with k
// contiguous (brs = 1, bcs = k), C dense column-major (crs = 1, ccs = m),
// m = n = k = 64 (checked by the dispatcher).
#pragma once
#include <cuda.h>

#include "sbt_common.cuh"
#include "sm100_ptx.cuh"

namespace sbt {
namespace small64 {

#ifndef SBT_SMALL64_G
#define SBT_SMALL64_G 1
#endif
constexpr int G = SBT_SMALL64_G;  // matrices per group (64 threads each)
constexpr int kThreads = 64 * G;
// one stage per CTA, six single-matrix CTAs per SM (12 warps): while some CTAs
// wait for their next matrix the others compute -- the FFMA pipe needs more
// than one warp per scheduler, which one 3-stage CTA of 4 warps could not
// provide (measured: 0.52 -> 0.62 -> 0.65 of HBM for 3-stage / 3 x 2-matrix /
// 6 x 1-matrix CTAs)
constexpr int STAGES = 1;
constexpr int CTAS_PER_SM = 6 / G;
constexpr int S = 64, LDB = 68;
constexpr int A_FLOATS = S * S, B_FLOATS = LDB * S;
constexpr int STAGE_FLOATS = G * (A_FLOATS + B_FLOATS);
constexpr int SMEM_BYTES = STAGES * STAGE_FLOATS * 4 + 64;

__global__ void __launch_bounds__(kThreads, CTAS_PER_SM)
small64_kernel(GemmParams<float> p, const __grid_constant__ CUtensorMap tmA,
               const __grid_constant__ CUtensorMap tmB, int64_t ngroups) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* sm = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + STAGES * STAGE_FLOATS * 4);
  const int tid = threadIdx.x;
  constexpr uint32_t TX = uint32_t(STAGE_FLOATS * 4);

  auto issue = [&](int64_t grp, int slot) {
    float* sa = sm + slot * STAGE_FLOATS;
    ptx::mbar_arrive_expect_tx(&full[slot], TX);
    ptx::tma_load_4d(sa, &tmA, &full[slot], 0, 0, int(grp * G), 0);
    ptx::tma_load_4d(sa + G * A_FLOATS, &tmB, &full[slot], 0, 0, int(grp * G), 0);
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

  const int mat = tid >> 6;             // matrix of the group
  const int lt = tid & 63;
  const int i0 = (lt & 7) * 8;          // 8 consecutive rows
  const int j0 = lt >> 3;               // columns j0, j0 + 8, ..., j0 + 56
  const bool vec = p.beta == 0.f && (p.cps % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(p.c) & 15) == 0);
  uint32_t it = 0;
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++it) {
    const int slot = int(it % STAGES);
    ptx::mbar_wait(&full[slot], (it / STAGES) & 1u);
    const int64_t bidx = grp * G + mat;
    if (bidx < p.batch) {
      const float* sa = sm + slot * STAGE_FLOATS + mat * A_FLOATS;
      const float* sb = sm + slot * STAGE_FLOATS + G * A_FLOATS + mat * B_FLOATS;
      float acc[8][8];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
#pragma unroll 2
      for (int l0 = 0; l0 < S; l0 += 4) {
        float4 bq[8];  // B(l0..l0+3, j0 + 8c)
#pragma unroll
        for (int c = 0; c < 8; ++c)
          bq[c] = *reinterpret_cast<const float4*>(sb + l0 + (j0 + 8 * c) * LDB);
#pragma unroll
        for (int dl = 0; dl < 4; ++dl) {
          const float4 a0 = *reinterpret_cast<const float4*>(sa + i0 + (l0 + dl) * S);
          const float4 a1 = *reinterpret_cast<const float4*>(sa + i0 + 4 + (l0 + dl) * S);
          const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float b = dl == 0 ? bq[c].x : dl == 1 ? bq[c].y : dl == 2 ? bq[c].z : bq[c].w;
#pragma unroll
            for (int r = 0; r < 8; ++r) acc[r][c] = fmaf(a[r], b, acc[r][c]);
          }
        }
      }
      float* C = p.c + bidx * p.cps;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float* dst = C + i0 + int64_t(j0 + 8 * c) * S;
        if (vec) {
          reinterpret_cast<float4*>(dst)[0] =
              make_float4(p.alpha * acc[0][c], p.alpha * acc[1][c], p.alpha * acc[2][c],
                          p.alpha * acc[3][c]);
          reinterpret_cast<float4*>(dst)[1] =
              make_float4(p.alpha * acc[4][c], p.alpha * acc[5][c], p.alpha * acc[6][c],
                          p.alpha * acc[7][c]);
        } else {
#pragma unroll
          for (int r = 0; r < 8; ++r) store_out(dst + r, acc[r][c], p.alpha, p.beta);
        }
      }
    }
    __syncthreads();  // the slot is free again
    const int64_t gnext = grp + int64_t(STAGES) * gridDim.x;
    if (tid == 0 && gnext < ngroups) issue(gnext, slot);
  }
}

}  // namespace small64
}  // namespace sbt

namespace sbt {
namespace small64mma {

// K3 (fp32, n = 32 / 64) on the tensor pipe: warp-level mma.sync m16n8k8 TF32
// with the 3xTF32 split (a_hi b_hi + a_hi b_lo + a_lo b_hi, round-to-nearest
// TF32 parts), fp32 register accumulators.  The register-blocked FFMA kernels
// are bound by shared-memory wavefronts at these sizes (ncu: LSU 76-79% busy);
// mma.sync TF32 runs at ~278 TFLOP/s on this part (measured), 93 TFLOP/s as
// 3xTF32.
//
// A CTA stage holds G matrices (one 3-D TMA box per operand); each matrix is
// computed by S / 16 warps of 16 C rows x S columns.  Two stages per CTA.  A
// lands as (LDA m) x S k and B as (LDB k) x S n, the TMA zero fill padding the
// rows so that both fragment patterns hit 32 distinct banks (LDA = 8 mod 32,
// LDB = 4 mod 32).  Operand contract as small64_kernel, at n = S.
template <int S>
struct Cfg {
  static constexpr int LDA = S + 8, LDB = S + 4;
  static constexpr int G = S == 64 ? 1 : 4;               // matrices per stage
  static constexpr int kWarps = G * (S / 16);
  static constexpr int kThreads = 32 * kWarps;
  static constexpr int STAGES = 2;
  static constexpr int CTAS_PER_SM = S == 64 ? 3 : 2;
  static constexpr int A_FLOATS = S * LDA, B_FLOATS = S * LDB;
  static constexpr int STAGE_FLOATS = G * (A_FLOATS + B_FLOATS);
  static constexpr int SMEM_BYTES = STAGES * STAGE_FLOATS * 4 + 64;
};
constexpr int LDA = Cfg<64>::LDA, LDB = Cfg<64>::LDB;   // (n = 64, for the launcher)

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4],
                                         const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int S>
__global__ void __launch_bounds__(Cfg<S>::kThreads, Cfg<S>::CTAS_PER_SM)
small_mma_kernel(GemmParams<float> p, const __grid_constant__ CUtensorMap tmA,
                 const __grid_constant__ CUtensorMap tmB, int64_t ngroups) {
  using C_ = Cfg<S>;
  constexpr int G = C_::G, STAGES = C_::STAGES, LDA_ = C_::LDA, LDB_ = C_::LDB;
  constexpr int NT8 = S / 8;                       // 8-wide N tiles = K steps
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* sm = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + STAGES * C_::STAGE_FLOATS * 4);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  constexpr uint32_t TX = uint32_t(C_::STAGE_FLOATS * 4);
  auto issue = [&](int64_t grp, int slot) {
    float* sa = sm + slot * C_::STAGE_FLOATS;
    ptx::mbar_arrive_expect_tx(&full[slot], TX);
    ptx::tma_load_4d(sa, &tmA, &full[slot], 0, 0, int(grp * G), 0);
    ptx::tma_load_4d(sa + G * C_::A_FLOATS, &tmB, &full[slot], 0, 0, int(grp * G), 0);
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
  const int mat = warp / (S / 16);                 // matrix of the group
  const int r0 = (warp % (S / 16)) * 16 + g;      // this lane's C rows r0, r0 + 8
  uint32_t it = 0;
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++it) {
    const int slot = int(it % STAGES);
    ptx::mbar_wait(&full[slot], (it / STAGES) & 1u);
    const int64_t bidx = grp * G + mat;
    const float* sa = sm + slot * C_::STAGE_FLOATS + mat * C_::A_FLOATS;   // A[m][k] at k*LDA + m
    const float* sb = sm + slot * C_::STAGE_FLOATS + G * C_::A_FLOATS +
                      mat * C_::B_FLOATS;                                  // B[k][n] at n*LDB + k
    float acc[NT8][4];
#pragma unroll
    for (int j = 0; j < NT8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    if (bidx < p.batch) {
#pragma unroll 2
      for (int k0 = 0; k0 < S; k0 += 8) {
        uint32_t ah[4], al[4];
        ptx::split_tf32(sa[(k0 + t) * LDA_ + r0], ah[0], al[0]);
        ptx::split_tf32(sa[(k0 + t) * LDA_ + r0 + 8], ah[1], al[1]);
        ptx::split_tf32(sa[(k0 + t + 4) * LDA_ + r0], ah[2], al[2]);
        ptx::split_tf32(sa[(k0 + t + 4) * LDA_ + r0 + 8], ah[3], al[3]);
#pragma unroll
        for (int j = 0; j < NT8; ++j) {
          uint32_t bh[2], bl[2];
          ptx::split_tf32(sb[(8 * j + g) * LDB_ + k0 + t], bh[0], bl[0]);
          ptx::split_tf32(sb[(8 * j + g) * LDB_ + k0 + t + 4], bh[1], bl[1]);
          mma_tf32(acc[j], al, bh);      // small cross terms first
          mma_tf32(acc[j], ah, bl);
          mma_tf32(acc[j], ah, bh);
        }
      }
    }
    __syncthreads();  // every warp has read the slot
    const int64_t gn = grp + int64_t(STAGES) * gridDim.x;
    if (tid == 0 && gn < ngroups) issue(gn, slot);
    if (bidx < p.batch) {
      float* C = p.c + bidx * p.cps;               // C[m][n] at m + n * S
#pragma unroll
      for (int j = 0; j < NT8; ++j) {
        const int n = 8 * j + 2 * t;
        store_out(C + r0 + int64_t(n) * S, acc[j][0], p.alpha, p.beta);
        store_out(C + r0 + int64_t(n + 1) * S, acc[j][1], p.alpha, p.beta);
        store_out(C + r0 + 8 + int64_t(n) * S, acc[j][2], p.alpha, p.beta);
        store_out(C + r0 + 8 + int64_t(n + 1) * S, acc[j][3], p.alpha, p.beta);
      }
    }
  }
}

}  // namespace small64mma
}  // namespace sbt
