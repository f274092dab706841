// K1/K2 (fp32): strided batched GEMM on the 5th-generation tensor cores with
// 3xTF32 (fp32-accurate) arithmetic: tcgen05.mma kind::tf32, TMEM accumulator.
//
//   C = alpha * (A_hi B_hi + A_hi B_lo + A_lo B_hi) + beta * C,   x = x_hi + x_lo
//
// The tensor core truncates fp32 operands to TF32, so x_hi is the raw fp32
// value and x_lo = x - trunc_tf32(x) (see k_tf32x3_pair_tma.cuh).
// 1xTF32 misses the reference's fp32 tolerance (~3e-4 vs 1e-5, SURVEY.md
// Appendix C); the three-term split reaches ~1e-7.
//
// Operands are read IN PLACE at their strides (no transpose, no copy).  Each
// operand tile is staged into a 128-byte-swizzled canonical UMMA layout whose
// major mode is the operand's unit-stride global mode:
//   A: acs == 1 -> K-major tile, ars == 1 -> MN-major tile   (op T / op N)
//   B: brs == 1 -> K-major tile, bcs == 1 -> MN-major tile   (op N / op T)
// so every op-flag combination the dispatcher produces is a native tensor-core
// operand (UMMA's a_major / b_major bits) -- the permutation is folded into the
// shared-memory staging, never materialised in HBM.
//
// This 1-CTA kernel serves skinny problems (N <= 128 after orientation, e.g.
// the rank-32 Tucker mode products); large tiles go to the CTA-pair kernel.
//
// Pipeline (one 128 x BN output tile per CTA, 9 warps):
//   warps 0-7 : producers.  16-byte coalesced LDG of the next K-block is in
//               flight while the current one is split into hi/lo TF32 in
//               registers and stored (STS.128) into the swizzled stage buffer;
//               fence.proxy.async + mbarrier arrive hands the stage to the MMA.
//               After the main loop the same warps drain TMEM (tcgen05.ld) and
//               store C with the reference's beta rule.
//   warp 8    : TMEM allocation and the single-thread tcgen05.mma issuer;
//               tcgen05.commit releases each stage back to the producers.
#pragma once
#include "sbt_common.cuh"
#include "sm100_ptx.cuh"

namespace sbt {
namespace tf32x3 {

constexpr int BM = 128;
constexpr int BK = 32;            // fp32 elements per K-block = one 128 B swizzle row
constexpr int kProducerWarps = 8;
constexpr int kProducers = kProducerWarps * 32;
constexpr int kThreads = kProducers + 32;

template <int BN>
struct Cfg {
  static constexpr int STAGES = BN == 256 ? 2 : BN == 128 ? 3 : BN == 64 ? 4 : 5;
  static constexpr int A_BYTES = BM * BK * 4;  // one of hi/lo
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int A_VEC = BM * BK / 4 / kProducers;  // float4 per producer thread
  static constexpr int B_VEC = BN * BK / 4 / kProducers;
  // main (hi*hi) accumulator + a separate one for the two small cross terms
  // (the tensor core truncates the fp32 accumulator on every MMA; keeping the
  // 2^-11-sized terms apart roughly halves that error, cf. k_tf32x3_pair_tma)
  static constexpr int ACC_COLS = BN < 32 ? 32 : BN;
  static constexpr int TMEM_COLS = 2 * ACC_COLS;
};

// Byte offset of element (mn, k) inside a [rows x 32] K-major SW128 tile.
__device__ __forceinline__ uint32_t kmajor_off(int mn, int kchunk) {
  return uint32_t(mn) * 128u + (uint32_t(kchunk ^ (mn & 7)) << 4);
}
// Byte offset of the 16 B chunk holding (mn4*4 .. mn4*4+3, k) in an MN-major
// SW128_BASE32B tile: 512 B atoms of 32 MN x 4 K, `mn_atoms` atoms per 4-deep
// K group, 32 B granule index XOR (k % 4).
__device__ __forceinline__ uint32_t mnmajor_off(int mn4, int k, int mn_atoms) {
  return uint32_t(((k >> 2) * mn_atoms + (mn4 >> 3)) * 512 + (k & 3) * 128 +
                  ((((mn4 >> 1) & 3) ^ (k & 3)) << 5) + ((mn4 & 1) << 4));
}

template <int BN, bool A_K, bool B_K>
__global__ void __launch_bounds__(kThreads, 1)
tf32x3_gemm_kernel(GemmParams<float> p, int64_t tiles_m, int64_t tiles_n) {
  using C_ = Cfg<BN>;
  constexpr int STAGES = C_::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C_::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* accf = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  // tile coordinates (m fastest: consecutive CTAs share the B tile in L2)
  int64_t t = blockIdx.x;
  const int64_t tm = t % tiles_m;
  t /= tiles_m;
  const int64_t tn = t % tiles_n;
  t /= tiles_n;
  const int64_t pb = t % p.batch;
  const int64_t qb = t / p.batch;
  const int64_t m0 = tm * BM, n0 = tn * BN;
  const float* __restrict__ A = p.a + pb * p.aps + qb * p.aps2;
  const float* __restrict__ B = p.b + pb * p.bps + qb * p.bps2;
  float* __restrict__ Cp = p.c + pb * p.cps + qb * p.cps2;
  const int nkb = int((p.k + BK - 1) / BK);

  if (warp == kProducerWarps) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        ptx::mbar_init(&full[s], kProducers);
        ptx::mbar_init(&empty[s], 1);
      }
      ptx::mbar_init(accf, 1);
      ptx::fence_mbarrier_init();
    }
    __syncwarp();
    ptx::tmem_alloc(tmem_slot, C_::TMEM_COLS);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < kProducerWarps) {
    // ------------------------------------------------------------ producers
    auto load = [&](int kb, float4 (&ra)[C_::A_VEC], float4 (&rb)[C_::B_VEC]) {
      const int64_t k0 = int64_t(kb) * BK;
#pragma unroll
      for (int i = 0; i < C_::A_VEC; ++i) {
        const int e = tid + i * kProducers;
        int64_t gm, gk;
        if (A_K) { gm = m0 + (e >> 3); gk = k0 + (e & 7) * 4; }
        else     { gk = k0 + (e >> 5); gm = m0 + (e & 31) * 4; }
        ra[i] = (gm < p.m && gk < p.k) ? ptx::ldg_nc_v4(A + gm * p.ars + gk * p.acs)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int i = 0; i < C_::B_VEC; ++i) {
        const int e = tid + i * kProducers;
        int64_t gn, gk;
        if (B_K) { gn = n0 + (e >> 3); gk = k0 + (e & 7) * 4; }
        else     { gk = k0 + e / (BN / 4); gn = n0 + (e % (BN / 4)) * 4; }
        rb[i] = (gn < p.n && gk < p.k) ? ptx::ldg_nc_v4(B + gk * p.brs + gn * p.bcs)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto produce = [&](int kb, const float4 (&ra)[C_::A_VEC], const float4 (&rb)[C_::B_VEC]) {
      const int s = kb % STAGES;
      ptx::mbar_wait(&empty[s], (uint32_t(kb / STAGES) & 1u) ^ 1u);
      uint8_t* st = smem + s * C_::STAGE_BYTES;
      const uint32_t a_hi = ptx::smem_addr(st);
      const uint32_t a_lo = a_hi + C_::A_BYTES;
      const uint32_t b_hi = a_lo + C_::A_BYTES;
      const uint32_t b_lo = b_hi + C_::B_BYTES;
#pragma unroll
      for (int i = 0; i < C_::A_VEC; ++i) {
        const int e = tid + i * kProducers;
        const uint32_t off = A_K ? kmajor_off(e >> 3, e & 7) : mnmajor_off(e & 31, e >> 5, BM / 32);
        uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
        ptx::split_tf32_fast(ra[i].x, h0, l0);
        ptx::split_tf32_fast(ra[i].y, h1, l1);
        ptx::split_tf32_fast(ra[i].z, h2, l2);
        ptx::split_tf32_fast(ra[i].w, h3, l3);
        ptx::sts_v4(a_hi + off, h0, h1, h2, h3);
        ptx::sts_v4(a_lo + off, l0, l1, l2, l3);
      }
#pragma unroll
      for (int i = 0; i < C_::B_VEC; ++i) {
        const int e = tid + i * kProducers;
        const uint32_t off = B_K ? kmajor_off(e >> 3, e & 7)
                                 : mnmajor_off(e % (BN / 4), e / (BN / 4), BN / 32);
        uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
        ptx::split_tf32_fast(rb[i].x, h0, l0);
        ptx::split_tf32_fast(rb[i].y, h1, l1);
        ptx::split_tf32_fast(rb[i].z, h2, l2);
        ptx::split_tf32_fast(rb[i].w, h3, l3);
        ptx::sts_v4(b_hi + off, h0, h1, h2, h3);
        ptx::sts_v4(b_lo + off, l0, l1, l2, l3);
      }
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&full[s]);
    };

    // ping-pong register sets: K-block kb+1 is in flight while kb is split/stored
    float4 ra0[C_::A_VEC], rb0[C_::B_VEC], ra1[C_::A_VEC], rb1[C_::B_VEC];
    load(0, ra0, rb0);
    for (int kb = 0; kb < nkb; kb += 2) {
      if (kb + 1 < nkb) load(kb + 1, ra1, rb1);
      produce(kb, ra0, rb0);
      if (kb + 1 >= nkb) break;
      if (kb + 2 < nkb) load(kb + 2, ra0, rb0);
      produce(kb + 1, ra1, rb1);
    }
  } else {
    // ------------------------------------------------------------ MMA issuer
    // warp-uniform loop, one elected lane issues (descriptors stay uniform)
    constexpr uint32_t idesc = ptx::idesc_tf32(BM, BN, !A_K, !B_K);
    // per-MMA (K = 8) descriptor advance: 32 B inside a K-major row, or one
    // 8-deep K group (SBO) for MN-major
    // K-major: one K=8 step = 32 B inside the 128 B swizzle row.
    // MN-major: one K=8 step = two 4-deep K groups (SBO each).
    constexpr uint32_t a_sbo = A_K ? 1024u : uint32_t(BM / 32) * 512u;
    constexpr uint32_t a_lbo = A_K ? 16u : 512u;
    constexpr uint32_t b_sbo = B_K ? 1024u : uint32_t(BN / 32) * 512u;
    constexpr uint32_t b_lbo = B_K ? 16u : 512u;
    constexpr uint32_t a_step = A_K ? 32u : 2u * a_sbo;
    constexpr uint32_t b_step = B_K ? 32u : 2u * b_sbo;
    constexpr uint32_t a_lay = A_K ? ptx::kLayoutSW128 : ptx::kLayoutSW128Base32B;
    constexpr uint32_t b_lay = B_K ? ptx::kLayoutSW128 : ptx::kLayoutSW128Base32B;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = uint32_t(kb / STAGES) & 1u;
      ptx::mbar_wait(&full[s], ph);
      ptx::tc_fence_after();
      const uint32_t a_hi = ptx::smem_addr(smem + s * C_::STAGE_BYTES);
      const uint32_t a_lo = a_hi + C_::A_BYTES;
      const uint32_t b_hi = a_lo + C_::A_BYTES;
      const uint32_t b_lo = b_hi + C_::B_BYTES;
      if (ptx::elect_one_sync()) {
#pragma unroll
        for (int j = 0; j < BK / 8; ++j) {
          const uint64_t dah = ptx::umma_desc(a_hi + j * a_step, a_lbo, a_sbo, a_lay);
          const uint64_t dal = ptx::umma_desc(a_lo + j * a_step, a_lbo, a_sbo, a_lay);
          const uint64_t dbh = ptx::umma_desc(b_hi + j * b_step, b_lbo, b_sbo, b_lay);
          const uint64_t dbl = ptx::umma_desc(b_lo + j * b_step, b_lbo, b_sbo, b_lay);
          const uint32_t acc = (kb | j) ? 1u : 0u;
          const uint32_t small = tmem_base + C_::ACC_COLS;
          ptx::mma_tf32_ss(small, dal, dbh, idesc, acc);  // small terms apart
          ptx::mma_tf32_ss(small, dah, dbl, idesc, 1u);
          ptx::mma_tf32_ss(tmem_base, dah, dbh, idesc, acc);
        }
        ptx::tc_commit(&empty[s]);  // stage reusable once these MMAs retire
      }
      __syncwarp();
    }
    if (ptx::elect_one_sync()) ptx::tc_commit(accf);  // accumulator complete
    __syncwarp();
  }

  // ------------------------------------------------------------ epilogue
  if (warp < kProducerWarps) {
    ptx::mbar_wait(accf, 0);
    ptx::tc_fence_after();
    const int quarter = warp & 3;
    constexpr int HALF = BN / 2;
    const int col0 = (warp >> 2) * HALF;
    const int64_t row = m0 + quarter * 32 + lane;
    const bool row_ok = row < p.m;
    float* crow = Cp + row * p.crs;
#pragma unroll 1
    for (int cc = 0; cc < HALF; cc += 16) {
      uint32_t r[16], q[16];
      const uint32_t ta = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(col0 + cc);
      ptx::tmem_ld16(ta, r);
      ptx::tmem_ld16(ta + C_::ACC_COLS, q);
      ptx::tmem_ld_wait();
      if (row_ok) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t col = n0 + col0 + cc + j;
          if (col < p.n)
            store_out(crow + col * p.ccs, __uint_as_float(r[j]) + __uint_as_float(q[j]), p.alpha,
                      p.beta);
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kProducerWarps) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, C_::TMEM_COLS);
  }
}

}  // namespace tf32x3
}  // namespace sbt
