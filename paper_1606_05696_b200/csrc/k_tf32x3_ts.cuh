// K1 (fp32), persistent variant: 3xTF32 strided batched GEMM with the A operand
// split into Tensor Memory and the B operand split into shared memory.
//
// Why: 3xTF32 issues three MMAs per K-step, so with both operands in shared
// memory the tensor core's smem reads (plus the producers' stores) exceed the
// SM's ~128 B/clk shared-memory bandwidth.  Staging A (hi and lo) in TMEM via
// tcgen05.st removes A from the smem traffic entirely; TMEM has its own
// datapath.  A persistent tile loop with two TMEM accumulators lets the
// epilogue of tile i overlap the main loop of tile i+1.
//
// TMEM (512 columns): [0, 2*BN) two fp32 accumulators (lane = row), then
// STAGES A stages of 64 columns (32 hi + 32 lo; lane = row, column = k).
//
// Warp roles (13 warps):
//   0-3   A producers: thread r owns tile row r; loads its 32 k-values of the
//         next K-block (coalesced along whichever of A's modes is unit
//         stride), splits hi/lo, tcgen05.st into the stage's TMEM columns.
//   4-7   epilogue: tcgen05.ld a finished accumulator, alpha/beta, store C.
//   8-11  B producers: 16-byte LDG, hi/lo split, STS into the 128 B swizzled
//         K-major (SW128) or MN-major (SW128_BASE32B) canonical layout.
//   12    TMEM allocator + single-thread tcgen05.mma issuer.
#pragma once
#include "sbt_common.cuh"
#include "sm100_ptx.cuh"

namespace sbt {
namespace tf32ts {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 32;
constexpr int STAGES = 4;
constexpr int kThreads = 13 * 32;
constexpr int B_STAGE_BYTES = 2 * BN * BK * 4;                    // hi + lo
constexpr int SMEM_BYTES = STAGES * B_STAGE_BYTES + 1024 + 256;
constexpr uint32_t kAccCols = 2 * BN;                              // 256
constexpr uint32_t kACol0 = kAccCols;                              // A stages start
constexpr int B_VEC = BN * BK / 4 / 128;                           // float4 per B thread (8)

__device__ __forceinline__ uint32_t kmajor_off(int mn, int kchunk) {
  return uint32_t(mn) * 128u + (uint32_t(kchunk ^ (mn & 7)) << 4);
}
__device__ __forceinline__ uint32_t mnmajor_off(int mn4, int k, int mn_atoms) {
  return uint32_t(((k >> 2) * mn_atoms + (mn4 >> 3)) * 512 + (k & 3) * 128 +
                  ((((mn4 >> 1) & 3) ^ (k & 3)) << 5) + ((mn4 & 1) << 4));
}

struct TileCoord {
  int64_t m0, n0, pb, qb;
};
__device__ __forceinline__ TileCoord tile_coord(int64_t t, int64_t tiles_m, int64_t tiles_n,
                                                int64_t batch) {
  TileCoord c;
  c.m0 = (t % tiles_m) * BM;
  t /= tiles_m;
  c.n0 = (t % tiles_n) * BN;
  t /= tiles_n;
  c.pb = t % batch;
  c.qb = t / batch;
  return c;
}

template <bool A_K, bool B_K>
__global__ void __launch_bounds__(kThreads, 1)
tf32x3_ts_kernel(GemmParams<float> p, int64_t tiles_m, int64_t tiles_n, int64_t total) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * B_STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int nkb = int((p.k + BK - 1) / BK);

  if (warp == 12) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        ptx::mbar_init(&full[s], 256);  // 128 A + 128 B producer threads
        ptx::mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        ptx::mbar_init(&acc_full[b], 1);
        ptx::mbar_init(&acc_empty[b], 128);
      }
      ptx::fence_mbarrier_init();
    }
    __syncwarp();
    ptx::tmem_alloc(tmem_slot, 512);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ------------------------------------------------ A producers -> TMEM
    const int r = tid;  // tile row
    const uint32_t lane_addr = uint32_t(warp * 32) << 16;
    const int64_t my_tiles = (total - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t n_iter = my_tiles * nkb;
    // loads for flat iteration g = (local tile g / nkb, K-block g % nkb)
    auto load = [&](int64_t g, float (&v)[32]) {
      if (g >= n_iter) return;
      const int64_t t = blockIdx.x + (g / nkb) * gridDim.x;
      const int kb = int(g % nkb);
      const TileCoord tc = tile_coord(t, tiles_m, tiles_n, p.batch);
      const int64_t gm = tc.m0 + r;
      const bool row_ok = gm < p.m;
      const float* __restrict__ arow =
          p.a + tc.pb * p.aps + tc.qb * p.aps2 + (row_ok ? gm : 0) * p.ars;
      const int64_t k0 = int64_t(kb) * BK;
      if (A_K) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t gk = k0 + 4 * i;
          float4 x = (row_ok && gk < p.k) ? ptx::ldg_nc_v4_l1(arow + gk)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
          v[4 * i] = x.x; v[4 * i + 1] = x.y; v[4 * i + 2] = x.z; v[4 * i + 3] = x.w;
        }
      } else {
        const float* base = arow + k0 * p.acs;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          v[i] = (row_ok && k0 + i < p.k) ? ptx::ldg_nc(base + int64_t(i) * p.acs) : 0.f;
      }
    };
    auto produce = [&](int64_t g, const float (&v)[32]) {
      if (g >= n_iter) return;
      const uint32_t s = uint32_t(g % STAGES);
      ptx::mbar_wait(&empty[s], (uint32_t(g / STAGES) & 1u) ^ 1u);
      ptx::tc_fence_after();
      const uint32_t col = tmem + lane_addr + kACol0 + s * 64;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) ptx::split_tf32(v[16 * h + i], hi[i], lo[i]);
        ptx::tmem_st16(col + 16 * h, hi);
        ptx::tmem_st16(col + 32 + 16 * h, lo);
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&full[s]);
    };
    float r0[32], r1[32], r2[32];
    load(0, r0);
    load(1, r1);
    for (int64_t g = 0; g < n_iter; g += 3) {
      load(g + 2, r2);
      produce(g, r0);
      load(g + 3, r0);
      produce(g + 1, r1);
      load(g + 4, r1);
      produce(g + 2, r2);
    }
  } else if (warp < 8) {
    // ------------------------------------------------ epilogue
    const int q = warp & 3;
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    uint32_t tcount = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x, ++tcount) {
      const TileCoord tc = tile_coord(t, tiles_m, tiles_n, p.batch);
      const uint32_t b = tcount & 1u;
      ptx::mbar_wait(&acc_full[b], (tcount >> 1) & 1u);
      ptx::tc_fence_after();
      const int64_t row = tc.m0 + q * 32 + lane;
      const bool row_ok = row < p.m;
      float* __restrict__ crow = p.c + tc.pb * p.cps + tc.qb * p.cps2 + (row_ok ? row : 0) * p.crs;
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
            float4 o = make_float4(p.alpha * __uint_as_float(v[j]), p.alpha * __uint_as_float(v[j + 1]),
                                   p.alpha * __uint_as_float(v[j + 2]), p.alpha * __uint_as_float(v[j + 3]));
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
      ptx::mbar_arrive(&acc_empty[b]);
    }
  } else if (warp < 12) {
    // ------------------------------------------------ B producers -> SMEM
    const int bt = tid - 256;  // 0..127
    const int64_t my_tiles = (total - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t n_iter = my_tiles * nkb;
    auto load = [&](int64_t g, float4 (&v)[B_VEC]) {
      if (g >= n_iter) return;
      const int64_t t = blockIdx.x + (g / nkb) * gridDim.x;
      const int kb = int(g % nkb);
      const TileCoord tc = tile_coord(t, tiles_m, tiles_n, p.batch);
      const float* __restrict__ B = p.b + tc.pb * p.bps + tc.qb * p.bps2;
      const int64_t k0 = int64_t(kb) * BK;
#pragma unroll
      for (int i = 0; i < B_VEC; ++i) {
        const int e = bt + i * 128;
        int64_t gn, gk;
        if (B_K) { gn = tc.n0 + (e >> 3); gk = k0 + (e & 7) * 4; }
        else     { gk = k0 + e / (BN / 4); gn = tc.n0 + (e % (BN / 4)) * 4; }
        v[i] = (gn < p.n && gk < p.k) ? ptx::ldg_nc_v4(B + gk * p.brs + gn * p.bcs)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto produce = [&](int64_t g, const float4 (&v)[B_VEC]) {
      if (g >= n_iter) return;
      const uint32_t s = uint32_t(g % STAGES);
      ptx::mbar_wait(&empty[s], (uint32_t(g / STAGES) & 1u) ^ 1u);
      const uint32_t b_hi = ptx::smem_addr(smem + s * B_STAGE_BYTES);
      const uint32_t b_lo = b_hi + BN * BK * 4;
#pragma unroll
      for (int i = 0; i < B_VEC; ++i) {
        const int e = bt + i * 128;
        const uint32_t off = B_K ? kmajor_off(e >> 3, e & 7)
                                 : mnmajor_off(e % (BN / 4), e / (BN / 4), BN / 32);
        uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
        ptx::split_tf32(v[i].x, h0, l0);
        ptx::split_tf32(v[i].y, h1, l1);
        ptx::split_tf32(v[i].z, h2, l2);
        ptx::split_tf32(v[i].w, h3, l3);
        ptx::sts_v4(b_hi + off, h0, h1, h2, h3);
        ptx::sts_v4(b_lo + off, l0, l1, l2, l3);
      }
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&full[s]);
    };
    float4 r0[B_VEC], r1[B_VEC], r2[B_VEC];
    load(0, r0);
    load(1, r1);
    for (int64_t g = 0; g < n_iter; g += 3) {
      load(g + 2, r2);
      produce(g, r0);
      load(g + 3, r0);
      produce(g + 1, r1);
      load(g + 4, r1);
      produce(g + 2, r2);
    }
  } else if (lane == 0) {
    // ------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = ptx::idesc_tf32(BM, BN, false, !B_K);
    constexpr uint32_t b_sbo = B_K ? 1024u : uint32_t(BN / 32) * 512u;
    constexpr uint32_t b_lbo = B_K ? 16u : 512u;
    constexpr uint32_t b_step = B_K ? 32u : 2u * b_sbo;
    constexpr uint32_t b_lay = B_K ? ptx::kLayoutSW128 : ptx::kLayoutSW128Base32B;
    uint32_t it = 0, tcount = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x, ++tcount) {
      const uint32_t b = tcount & 1u;
      ptx::mbar_wait(&acc_empty[b], ((tcount >> 1) & 1u) ^ 1u);
      ptx::tc_fence_after();
      const uint32_t d = tmem + b * BN;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const uint32_t s = it % STAGES;
        ptx::mbar_wait(&full[s], (it / STAGES) & 1u);
        ptx::tc_fence_after();
        const uint32_t b_hi = ptx::smem_addr(smem + s * B_STAGE_BYTES);
        const uint32_t b_lo = b_hi + BN * BK * 4;
        const uint32_t a_col = tmem + kACol0 + s * 64;
#pragma unroll
        for (int j = 0; j < BK / 8; ++j) {
          const uint64_t dbh = ptx::umma_desc(b_hi + j * b_step, b_lbo, b_sbo, b_lay);
          const uint64_t dbl = ptx::umma_desc(b_lo + j * b_step, b_lbo, b_sbo, b_lay);
          const uint32_t ah = a_col + j * 8, al = a_col + 32 + j * 8;
          ptx::mma_tf32_ts(d, al, dbh, idesc, (kb | j) ? 1u : 0u);  // small terms first
          ptx::mma_tf32_ts(d, ah, dbl, idesc, 1u);
          ptx::mma_tf32_ts(d, ah, dbh, idesc, 1u);
        }
        ptx::tc_commit(&empty[s]);
      }
      ptx::tc_commit(&acc_full[b]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 12) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace tf32ts
}  // namespace sbt
