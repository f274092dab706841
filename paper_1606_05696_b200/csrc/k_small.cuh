// K3: small-matrix batched GEMM (every extent <= S, S in {8, 16, 32, 64}) for
// batches of 10^4 - 10^6 independent products (BASELINE configs[2]).
//
// The regime is HBM-bound for n <= 32 (fp32 AI = n/6 flop/B), so the kernel is
// a streaming pipeline: persistent CTAs walk groups of G = 4096 / S^2 batch
// entries.  A group's A and B matrices land in shared memory by TMA bulk copies
// (cp.async.bulk, one instruction per contiguous run -- the whole group when
// the batch is packed) STAGES groups ahead, completion counted on an mbarrier,
// so the SM keeps ~100 KB in flight with no load instructions on the compute
// warps.  Each thread multiplies a 4x4 output block from shared memory and
// writes it with 16-byte stores.
#pragma once
#include "sbt_common.cuh"
#include "sm100_ptx.cuh"

namespace sbt {
namespace small {

constexpr int kThreads = 256;
constexpr int STAGES = 3;  // fp32: 96 KB -> 2 CTAs/SM; fp64: 192 KB -> 1 CTA/SM

template <int S>
struct Shape {
  static constexpr int G = (4096 / (S * S)) > 0 ? 4096 / (S * S) : 1;  // matrices per group
  static constexpr int TPM = kThreads / G;                            // threads per matrix
  static constexpr int BPR = S / 4;                                   // 4x4 blocks per row
};

template <typename T, int S>
constexpr int stage_elems() { return 2 * Shape<S>::G * S * S; }
template <typename T, int S>
constexpr int smem_bytes() { return STAGES * stage_elems<T, S>() * int(sizeof(T)) + 64; }

// A_M: A stored with rows contiguous (ars == 1, acs == m), else (ars == k, acs == 1).
// B_K: B stored with k contiguous (brs == 1, bcs == k), else (brs == n, bcs == 1).
// C is dense with crs == 1, ccs == m.  Requires m*k and k*n multiples of 16 B
// and 16 B aligned batch strides (checked by the dispatcher).
template <typename T, int S, bool A_M, bool B_K>
__global__ void __launch_bounds__(kThreads)
small_batched_kernel(GemmParams<T> p, int64_t ngroups) {
  using Sh = Shape<S>;
  constexpr int G = Sh::G;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + STAGES * stage_elems<T, S>() * sizeof(T));
  const int tid = threadIdx.x;
  const int m = int(p.m), n = int(p.n), k = int(p.k);
  const int a_elems = m * k, b_elems = k * n;
  const int64_t total = p.batch;
  const bool a_contig = p.aps == a_elems, b_contig = p.bps == b_elems;

  // smem per stage: G matrices of A at stride a_elems, then G of B
  auto issue = [&](int64_t grp, int slot) {
    T* sa = sm + slot * stage_elems<T, S>();
    T* sb = sa + G * S * S;
    const int64_t b0 = grp * G;
    const int nmat = int(total - b0 < G ? total - b0 : G);
    if (tid == 0)
      ptx::mbar_arrive_expect_tx(&full[slot],
                                 uint32_t(nmat * (a_elems + b_elems) * int(sizeof(T))));
    __syncwarp();
    if (a_contig) {
      if (tid == 0) ptx::bulk_load(sa, p.a + b0 * p.aps, nmat * a_elems * sizeof(T), &full[slot]);
    } else if (tid < nmat) {
      ptx::bulk_load(sa + tid * a_elems, p.a + (b0 + tid) * p.aps, a_elems * sizeof(T), &full[slot]);
    }
    if (b_contig) {
      if (tid == 32) ptx::bulk_load(sb, p.b + b0 * p.bps, nmat * b_elems * sizeof(T), &full[slot]);
    } else if (tid >= 32 && tid < 32 + nmat) {
      ptx::bulk_load(sb + (tid - 32) * b_elems, p.b + (b0 + tid - 32) * p.bps,
                     b_elems * sizeof(T), &full[slot]);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) ptx::mbar_init(&full[s], 1);
    ptx::fence_mbarrier_init();
  }
  __syncthreads();

  const int g_local = tid / Sh::TPM;
  const int lt = tid - g_local * Sh::TPM;
  const int i0 = (lt % Sh::BPR) * 4, j0 = (lt / Sh::BPR) * 4;
  const bool vec_store = (m % 4 == 0) && (p.cps % 4 == 0) && p.beta == T(0) &&
                         ((reinterpret_cast<uintptr_t>(p.c) & 15) == 0);

  if (tid < 64) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      const int64_t gi = blockIdx.x + int64_t(s) * gridDim.x;
      if (gi < ngroups) issue(gi, s);
    }
  }
  uint32_t it = 0;
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++it) {
    const int slot = int(it % STAGES);
    ptx::mbar_wait(&full[slot], (it / STAGES) & 1u);
    const T* sa = sm + slot * stage_elems<T, S>() + g_local * a_elems;
    const T* sb = sm + slot * stage_elems<T, S>() + G * S * S + g_local * b_elems;
    const int64_t bidx = grp * G + g_local;
    if (bidx < total && i0 < m && j0 < n) {
      T acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = T(0);
#pragma unroll 4
      for (int l = 0; l < k; ++l) {
        T a[4], b[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) a[r] = A_M ? sa[(i0 + r) + l * m] : sa[(i0 + r) * k + l];
#pragma unroll
        for (int c = 0; c < 4; ++c) b[c] = B_K ? sb[l + (j0 + c) * k] : sb[l * n + j0 + c];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
      }
      T* C = p.c + bidx * p.cps;
      if (vec_store) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (j0 + c >= n) continue;
          T* dst = C + i0 + int64_t(j0 + c) * m;
          if constexpr (sizeof(T) == 4) {
            *reinterpret_cast<float4*>(dst) = make_float4(
                p.alpha * acc[0][c], p.alpha * acc[1][c], p.alpha * acc[2][c], p.alpha * acc[3][c]);
          } else {
            reinterpret_cast<double2*>(dst)[0] = make_double2(p.alpha * acc[0][c], p.alpha * acc[1][c]);
            reinterpret_cast<double2*>(dst)[1] = make_double2(p.alpha * acc[2][c], p.alpha * acc[3][c]);
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (j0 + c >= n) continue;
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (i0 + r < m) store_out(C + (i0 + r) + int64_t(j0 + c) * m, acc[r][c], p.alpha, p.beta);
        }
      }
    }
    __syncthreads();  // every thread is done with this slot
    const int64_t gnext = grp + int64_t(STAGES) * gridDim.x;
    if (tid < 64 && gnext < ngroups) issue(gnext, slot);
  }
}

}  // namespace small
}  // namespace sbt
