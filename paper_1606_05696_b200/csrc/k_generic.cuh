// K4: generic strided batched GEMM (SIMT FFMA / DFMA), correct for ANY strides.
//
// This is the fallback for requests the tensor-core kernels cannot take (odd
// extents, strides that are not 16-byte multiples, the reference's acceptance
// extents 1..8, test_acceptance.py:70).  Each CTA owns one BM x BN output tile
// of one (p, q) batch entry; tiles are visited grid-stride so any batch count
// (up to 10^6 and beyond, 64-bit indexing) fits one launch.
//
// Operand staging: each operand tile is read with the thread index running
// along whichever of its two global modes has the smaller stride, so unit
// stride operands load coalesced whatever the op flag (N/T) or extended
// layout; smem holds A as [BK][BM] and B as [BK][BN].
// Accumulation: one accumulator per output element, k ascending, fma chain --
// a fixed order per element, independent of tiling and batch split.
#pragma once
#include "sbt_common.cuh"

namespace sbt {

template <typename T, int BM, int BN, int BK, int TM, int TN>
struct GenericCfg {
  static constexpr int TX = BM / TM;  // threads along M (interleaved rows)
  static constexpr int TY = BN / TN;  // threads along N (blocked columns)
  static constexpr int NT = TX * TY;
  static constexpr int A_PER = BM * BK / NT;
  static constexpr int B_PER = BK * BN / NT;
  static constexpr int PAD = (sizeof(T) == 4) ? 4 : 2;
  static_assert(BM * BK % NT == 0 && BK * BN % NT == 0, "tile/threads mismatch");
};

template <typename T, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__(GenericCfg<T, BM, BN, BK, TM, TN>::NT)
generic_gemm_kernel(GemmParams<T> p, int64_t tiles_m, int64_t tiles_n, int64_t total_tiles,
                    int a_m_fast, int b_k_fast) {
  using Cfg = GenericCfg<T, BM, BN, BK, TM, TN>;
  constexpr int NT = Cfg::NT;
  __shared__ __align__(16) T As[BK][BM + Cfg::PAD];
  __shared__ __align__(16) T Bs[BK][BN + Cfg::PAD];

  const int tid = threadIdx.x;
  const int tx = tid % Cfg::TX;
  const int ty = tid / Cfg::TX;

  for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
    int64_t r = t;
    const int64_t tm = r % tiles_m;
    r /= tiles_m;
    const int64_t tn = r % tiles_n;
    r /= tiles_n;
    const int64_t pb = r % p.batch;
    const int64_t qb = r / p.batch;
    const int64_t m0 = tm * BM, n0 = tn * BN;
    const T* __restrict__ A = p.a + pb * p.aps + qb * p.aps2;
    const T* __restrict__ B = p.b + pb * p.bps + qb * p.bps2;

    T acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

    T ra[Cfg::A_PER], rb[Cfg::B_PER];
    auto load_tiles = [&](int64_t k0) {
#pragma unroll
      for (int e = 0; e < Cfg::A_PER; ++e) {
        const int idx = tid + e * NT;
        const int i = a_m_fast ? (idx % BM) : (idx / BK);
        const int l = a_m_fast ? (idx / BM) : (idx % BK);
        const int64_t gi = m0 + i, gl = k0 + l;
        ra[e] = (gi < p.m && gl < p.k) ? A[gi * p.ars + gl * p.acs] : T(0);
      }
#pragma unroll
      for (int e = 0; e < Cfg::B_PER; ++e) {
        const int idx = tid + e * NT;
        const int l = b_k_fast ? (idx % BK) : (idx / BN);
        const int j = b_k_fast ? (idx / BK) : (idx % BN);
        const int64_t gl = k0 + l, gj = n0 + j;
        rb[e] = (gl < p.k && gj < p.n) ? B[gl * p.brs + gj * p.bcs] : T(0);
      }
    };
    auto store_tiles = [&]() {
#pragma unroll
      for (int e = 0; e < Cfg::A_PER; ++e) {
        const int idx = tid + e * NT;
        const int i = a_m_fast ? (idx % BM) : (idx / BK);
        const int l = a_m_fast ? (idx / BM) : (idx % BK);
        As[l][i] = ra[e];
      }
#pragma unroll
      for (int e = 0; e < Cfg::B_PER; ++e) {
        const int idx = tid + e * NT;
        const int l = b_k_fast ? (idx % BK) : (idx / BN);
        const int j = b_k_fast ? (idx / BK) : (idx % BN);
        Bs[l][j] = rb[e];
      }
    };

    load_tiles(0);
    for (int64_t k0 = 0; k0 < p.k; k0 += BK) {
      __syncthreads();  // previous compute done with smem
      store_tiles();
      __syncthreads();
      if (k0 + BK < p.k) load_tiles(k0 + BK);  // prefetch overlaps the math below
#pragma unroll
      for (int l = 0; l < BK; ++l) {
        T av[TM], bv[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) av[i] = As[l][tx + i * Cfg::TX];
#pragma unroll
        for (int j = 0; j < TN; ++j) bv[j] = Bs[l][ty * TN + j];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
      }
    }

    T* C = p.c + pb * p.cps + qb * p.cps2;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t gj = n0 + ty * TN + j;
      if (gj >= p.n) continue;
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int64_t gi = m0 + tx + i * Cfg::TX;
        if (gi < p.m) store_out(C + gi * p.crs + gj * p.ccs, acc[i][j], p.alpha, p.beta);
      }
    }
  }
}

}  // namespace sbt
