// K1 (fp32), CTA-pair variant: 3xTF32 strided batched GEMM on
// tcgen05.mma.cta_group::2 (UMMA M = 256, N = 256) with persistent tiles.
//
// A CTA pair (cluster of 2 on one TPC) computes a 256 x 256 output tile.  Each
// CTA stages its own 128 rows of A and HALF of B's 256 columns (hi and lo,
// 128 B swizzled canonical layouts); the leader's single MMA thread issues
// M=256 MMAs that read both CTAs' shared memory.  Per SM this halves the
// tensor core's B reads and the B split/store work relative to a 1-CTA tile,
// which is what keeps 3xTF32 (three MMAs per K-step) under the SM's
// shared-memory bandwidth.
//
// Synchronisation:
//   full[s]      leader smem, 2 x 256 producer arrivals (peer arrives remotely
//                with release.cluster after fence.proxy.async of its STS)
//   empty[s]     both CTAs, count 1: leader's tcgen05.commit multicast
//   acc_full[b]  both CTAs, count 1: multicast commit after a tile's last MMA
//   acc_empty[b] leader smem, 2 x 128 epilogue arrivals (peer remote)
// TMEM (per CTA, allocated pairwise): two 256-column fp32 accumulators.
//
// Warp roles per CTA (13 warps): 0-3 epilogue (TMEM lane quarters), 4-11
// producers (LDG.128 -> hi/lo split -> STS), 12 TMEM allocator (+ MMA issuer
// on the leader).
#pragma once
#include "sbt_common.cuh"
#include "sm100_ptx.cuh"

namespace sbt {
namespace tf32pair {

constexpr int BM = 256;        // pair tile rows (128 per CTA)
constexpr int BN = 256;        // pair tile cols (128 of B staged per CTA)
constexpr int HM = 128;        // rows per CTA
constexpr int HN = 128;        // B columns per CTA
constexpr int BK = 32;
constexpr int STAGES = 3;
constexpr int kThreads = 13 * 32;
constexpr int kProducers = 256;
constexpr int A_BYTES = HM * BK * 4;
constexpr int B_BYTES = HN * BK * 4;
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;             // 64 KB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int VEC = HM * BK / 4 / kProducers;                     // 4 float4 per operand

__device__ __forceinline__ uint32_t kmajor_off(int mn, int kchunk) {
  return uint32_t(mn) * 128u + (uint32_t(kchunk ^ (mn & 7)) << 4);
}
__device__ __forceinline__ uint32_t mnmajor_off(int mn4, int k, int mn_atoms) {
  return uint32_t(((k >> 2) * mn_atoms + (mn4 >> 3)) * 512 + (k & 3) * 128 +
                  ((((mn4 >> 1) & 3) ^ (k & 3)) << 5) + ((mn4 & 1) << 4));
}

struct Tile {
  int64_t m0, n0, pb, qb;
};
__device__ __forceinline__ Tile tile_of(int64_t t, int64_t tiles_m, int64_t tiles_n, int64_t batch) {
  Tile c;
  c.m0 = (t % tiles_m) * BM;
  t /= tiles_m;
  c.n0 = (t % tiles_n) * BN;
  t /= tiles_n;
  c.pb = t % batch;
  c.qb = t / batch;
  return c;
}

template <bool A_K, bool B_K>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
tf32x3_pair_kernel(GemmParams<float> p, int64_t tiles_m, int64_t tiles_n, int64_t total) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const uint32_t rank = ptx::cluster_rank();
  const bool leader = rank == 0;
  const int64_t pair = blockIdx.x >> 1;
  const int64_t npairs = gridDim.x >> 1;
  const int nkb = int((p.k + BK - 1) / BK);

  if (warp == 12) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        ptx::mbar_init(&full[s], 2 * kProducers);
        ptx::mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        ptx::mbar_init(&acc_full[b], 1);
        ptx::mbar_init(&acc_empty[b], 2 * 128);
      }
      ptx::fence_mbarrier_init();
    }
    __syncwarp();
    ptx::tmem_alloc2(tmem_slot, 512);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barriers initialised and TMEM allocated in both CTAs
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 4 && warp < 12) {
    // ------------------------------------------------------------ producers
    const int pt = tid - 128;  // 0..255
    uint32_t full_remote[STAGES];
#pragma unroll
    for (int s = 0; s < STAGES; ++s) full_remote[s] = ptx::mapa(&full[s], 0);
    const int64_t my_tiles = (total - pair + npairs - 1) / npairs;
    const int64_t n_iter = my_tiles * nkb;
    auto load = [&](int64_t g, float4 (&ra)[VEC], float4 (&rb)[VEC]) {
      if (g >= n_iter) return;
      const Tile tc = tile_of(pair + (g / nkb) * npairs, tiles_m, tiles_n, p.batch);
      const int64_t k0 = int64_t(g % nkb) * BK;
      const int64_t mb = tc.m0 + rank * HM, nb = tc.n0 + rank * HN;
      const float* __restrict__ A = p.a + tc.pb * p.aps + tc.qb * p.aps2;
      const float* __restrict__ B = p.b + tc.pb * p.bps + tc.qb * p.bps2;
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        const int e = pt + i * kProducers;
        int64_t gm, gk;
        if (A_K) { gm = mb + (e >> 3); gk = k0 + (e & 7) * 4; }
        else     { gk = k0 + (e >> 5); gm = mb + (e & 31) * 4; }
        ra[i] = (gm < p.m && gk < p.k) ? ptx::ldg_nc_v4(A + gm * p.ars + gk * p.acs)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
        int64_t gn, gk2;
        if (B_K) { gn = nb + (e >> 3); gk2 = k0 + (e & 7) * 4; }
        else     { gk2 = k0 + (e >> 5); gn = nb + (e & 31) * 4; }
        rb[i] = (gn < p.n && gk2 < p.k) ? ptx::ldg_nc_v4(B + gk2 * p.brs + gn * p.bcs)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto put = [](uint32_t hi_base, uint32_t lo_base, uint32_t off, const float4& v) {
      uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
      ptx::split_tf32(v.x, h0, l0);
      ptx::split_tf32(v.y, h1, l1);
      ptx::split_tf32(v.z, h2, l2);
      ptx::split_tf32(v.w, h3, l3);
      ptx::sts_v4(hi_base + off, h0, h1, h2, h3);
      ptx::sts_v4(lo_base + off, l0, l1, l2, l3);
    };
    auto produce = [&](int64_t g, const float4 (&ra)[VEC], const float4 (&rb)[VEC]) {
      if (g >= n_iter) return;
      const uint32_t s = uint32_t(g % STAGES);
      ptx::mbar_wait(&empty[s], (uint32_t(g / STAGES) & 1u) ^ 1u);
      const uint32_t a_hi = ptx::smem_addr(smem + s * STAGE_BYTES);
      const uint32_t a_lo = a_hi + A_BYTES;
      const uint32_t b_hi = a_lo + A_BYTES;
      const uint32_t b_lo = b_hi + B_BYTES;
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        const int e = pt + i * kProducers;
        put(a_hi, a_lo, A_K ? kmajor_off(e >> 3, e & 7) : mnmajor_off(e & 31, e >> 5, HM / 32),
            ra[i]);
        put(b_hi, b_lo, B_K ? kmajor_off(e >> 3, e & 7) : mnmajor_off(e & 31, e >> 5, HN / 32),
            rb[i]);
      }
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive_cluster(full_remote[s]);
    };
    float4 a0[VEC], b0[VEC], a1[VEC], b1[VEC];
    load(0, a0, b0);
    for (int64_t g = 0; g < n_iter; g += 2) {
      load(g + 1, a1, b1);
      produce(g, a0, b0);
      load(g + 2, a0, b0);
      produce(g + 1, a1, b1);
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp;
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    const uint32_t acc_empty_remote0 = ptx::mapa(&acc_empty[0], 0);
    const uint32_t acc_empty_remote1 = ptx::mapa(&acc_empty[1], 0);
    uint32_t tcount = 0;
    for (int64_t t = pair; t < total; t += npairs, ++tcount) {
      const Tile tc = tile_of(t, tiles_m, tiles_n, p.batch);
      const uint32_t b = tcount & 1u;
      ptx::mbar_wait(&acc_full[b], (tcount >> 1) & 1u);
      ptx::tc_fence_after();
      const int64_t row = tc.m0 + rank * HM + q * 32 + lane;
      const bool row_ok = row < p.m;
      float* __restrict__ crow =
          p.c + tc.pb * p.cps + tc.qb * p.cps2 + (row_ok ? row : 0) * p.crs;
      const bool vec = (p.ccs == 1) && ((reinterpret_cast<uintptr_t>(crow) & 15) == 0) &&
                       (tc.n0 + BN <= p.n) && p.beta == 0.f;
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 16) {
        uint32_t v[16];
        ptx::tmem_ld16(tmem + lane_addr + b * BN + cc, v);
        ptx::tmem_ld_wait();
        if (!row_ok) continue;
        if (vec) {
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            float4 o = make_float4(p.alpha * __uint_as_float(v[j]),
                                   p.alpha * __uint_as_float(v[j + 1]),
                                   p.alpha * __uint_as_float(v[j + 2]),
                                   p.alpha * __uint_as_float(v[j + 3]));
            *reinterpret_cast<float4*>(crow + tc.n0 + cc + j) = o;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int64_t col = tc.n0 + cc + j;
            if (col < p.n) store_out(crow + col * p.ccs, __uint_as_float(v[j]), p.alpha, p.beta);
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive_cluster(b ? acc_empty_remote1 : acc_empty_remote0);
    }
  } else if (leader && lane == 0) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = ptx::idesc_tf32(BM, BN, !A_K, !B_K);
    constexpr uint32_t a_sbo = A_K ? 1024u : uint32_t(HM / 32) * 512u;
    constexpr uint32_t a_lbo = A_K ? 16u : 512u;
    constexpr uint32_t b_sbo = B_K ? 1024u : uint32_t(HN / 32) * 512u;
    constexpr uint32_t b_lbo = B_K ? 16u : 512u;
    constexpr uint32_t a_step = A_K ? 32u : 2u * a_sbo;
    constexpr uint32_t b_step = B_K ? 32u : 2u * b_sbo;
    constexpr uint32_t a_lay = A_K ? ptx::kLayoutSW128 : ptx::kLayoutSW128Base32B;
    constexpr uint32_t b_lay = B_K ? ptx::kLayoutSW128 : ptx::kLayoutSW128Base32B;
    uint32_t it = 0, tcount = 0;
    for (int64_t t = pair; t < total; t += npairs, ++tcount) {
      const uint32_t b = tcount & 1u;
      ptx::mbar_wait_cluster(&acc_empty[b], ((tcount >> 1) & 1u) ^ 1u);
      ptx::tc_fence_after();
      const uint32_t d = tmem + b * BN;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const uint32_t s = it % STAGES;
        ptx::mbar_wait_cluster(&full[s], (it / STAGES) & 1u);
        ptx::tc_fence_after();
        const uint32_t a_hi = ptx::smem_addr(smem + s * STAGE_BYTES);
        const uint32_t a_lo = a_hi + A_BYTES;
        const uint32_t b_hi = a_lo + A_BYTES;
        const uint32_t b_lo = b_hi + B_BYTES;
#pragma unroll
        for (int j = 0; j < BK / 8; ++j) {
          const uint64_t dah = ptx::umma_desc(a_hi + j * a_step, a_lbo, a_sbo, a_lay);
          const uint64_t dal = ptx::umma_desc(a_lo + j * a_step, a_lbo, a_sbo, a_lay);
          const uint64_t dbh = ptx::umma_desc(b_hi + j * b_step, b_lbo, b_sbo, b_lay);
          const uint64_t dbl = ptx::umma_desc(b_lo + j * b_step, b_lbo, b_sbo, b_lay);
          ptx::mma2_tf32_ss(d, dal, dbh, idesc, (kb | j) ? 1u : 0u);
          ptx::mma2_tf32_ss(d, dah, dbl, idesc, 1u);
          ptx::mma2_tf32_ss(d, dah, dbh, idesc, 1u);
        }
        ptx::tc_commit2_mc(&empty[s], 0x3);
      }
      ptx::tc_commit2_mc(&acc_full[b], 0x3);
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();  // nobody leaves while the pair may still touch its smem / TMEM
  if (warp == 12) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem, 512);
  }
}

}  // namespace tf32pair
}  // namespace sbt
