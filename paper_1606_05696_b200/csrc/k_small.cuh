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

// four consecutive elements from a 16-byte aligned smem address
__device__ __forceinline__ void load4(const float* p, float& a, float& b, float& c, float& d) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  a = v.x; b = v.y; c = v.z; d = v.w;
}
__device__ __forceinline__ void load4(const double* p, double& a, double& b, double& c,
                                      double& d) {
  const double2 v0 = reinterpret_cast<const double2*>(p)[0];
  const double2 v1 = reinterpret_cast<const double2*>(p)[1];
  a = v0.x; b = v0.y; c = v1.x; d = v1.y;
}

template <int S>
struct Shape {
  static constexpr int G = (4096 / (S * S)) > 0 ? 4096 / (S * S) : 1;  // matrices per group
  static constexpr int TPM = kThreads / G;                            // threads per matrix
  static constexpr int BPR = S / 4;                                   // 4x4 blocks per row
};

// per-matrix smem slot: S*S elements + 32 B of padding, so that the G matrices
// of a group start on different banks (conflict-free 16-byte fragment loads)
template <typename T, int S>
__host__ __device__ constexpr int slot_elems() { return S * S + 32 / int(sizeof(T)); }
template <typename T, int S>
__host__ __device__ constexpr int stage_elems() { return 2 * Shape<S>::G * slot_elems<T, S>(); }
template <typename T, int S>
__host__ __device__ constexpr int smem_bytes() { return STAGES * stage_elems<T, S>() * int(sizeof(T)) + 64; }

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
  constexpr int SL = slot_elems<T, S>();

  // smem per stage: G padded matrix slots of A, then G of B; one bulk copy per
  // matrix and operand, issued by G threads in parallel
  auto issue = [&](int64_t grp, int slot) {
    T* sa = sm + slot * stage_elems<T, S>();
    T* sb = sa + G * SL;
    const int64_t b0 = grp * G;
    const int nmat = int(total - b0 < G ? total - b0 : G);
    if (tid == 0)
      ptx::mbar_arrive_expect_tx(&full[slot],
                                 uint32_t(nmat * (a_elems + b_elems) * int(sizeof(T))));
    __syncthreads();  // expect_tx precedes every completion of this phase
    if (tid < nmat)
      ptx::bulk_load(sa + tid * SL, p.a + (b0 + tid) * p.aps, a_elems * sizeof(T), &full[slot]);
    else if (tid >= 128 && tid < 128 + nmat)
      ptx::bulk_load(sb + (tid - 128) * SL, p.b + (b0 + tid - 128) * p.bps, b_elems * sizeof(T),
                     &full[slot]);
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) ptx::mbar_init(&full[s], 1);
    ptx::fence_mbarrier_init();
  }
  __syncthreads();

  const int g_local = tid / Sh::TPM;
  const int lt = tid - g_local * Sh::TPM;
  const int i0 = (lt % Sh::BPR) * 4, j0 = (lt / Sh::BPR) * 4;
  const bool vec4 = (m % 4 == 0) && (n % 4 == 0) && (k % 4 == 0);
  const bool vec_store = (m % 4 == 0) && (p.cps % 4 == 0) && p.beta == T(0) &&
                         ((reinterpret_cast<uintptr_t>(p.c) & 15) == 0);

#pragma unroll
  for (int s = 0; s < STAGES; ++s) {
    const int64_t gi = blockIdx.x + int64_t(s) * gridDim.x;
    if (gi < ngroups) issue(gi, s);
  }
  uint32_t it = 0;
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++it) {
    const int slot = int(it % STAGES);
    ptx::mbar_wait(&full[slot], (it / STAGES) & 1u);
    const T* sa = sm + slot * stage_elems<T, S>() + g_local * SL;
    const T* sb = sm + slot * stage_elems<T, S>() + G * SL + g_local * SL;
    const int64_t bidx = grp * G + g_local;
    if (bidx < total && i0 < m && j0 < n) {
      T acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = T(0);
      if (vec4) {
        // 4-deep k chunks: 4 + 4 sixteen-byte-aligned quads -> 64 FMA
        for (int l0 = 0; l0 < k; l0 += 4) {
          T a[4][4], b[4][4];  // a[r][dl] = A(i0+r, l0+dl), b[dl][c] = B(l0+dl, j0+c)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (A_M) load4(sa + i0 + (l0 + q) * m, a[0][q], a[1][q], a[2][q], a[3][q]);
            else     load4(sa + (i0 + q) * k + l0, a[q][0], a[q][1], a[q][2], a[q][3]);
            if (B_K) load4(sb + l0 + (j0 + q) * k, b[0][q], b[1][q], b[2][q], b[3][q]);
            else     load4(sb + (l0 + q) * n + j0, b[q][0], b[q][1], b[q][2], b[q][3]);
          }
#pragma unroll
          for (int dl = 0; dl < 4; ++dl)
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int c = 0; c < 4; ++c) acc[r][c] = fma(a[r][dl], b[dl][c], acc[r][c]);
        }
      } else {
        for (int l = 0; l < k; ++l) {
          T a[4], b[4];
#pragma unroll
          for (int r = 0; r < 4; ++r)
            a[r] = (i0 + r < m) ? (A_M ? sa[(i0 + r) + l * m] : sa[(i0 + r) * k + l]) : T(0);
#pragma unroll
          for (int c = 0; c < 4; ++c)
            b[c] = (j0 + c < n) ? (B_K ? sb[l + (j0 + c) * k] : sb[l * n + j0 + c]) : T(0);
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
        }
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
    if (gnext < ngroups) issue(gnext, slot);
  }
}

}  // namespace small
}  // namespace sbt
