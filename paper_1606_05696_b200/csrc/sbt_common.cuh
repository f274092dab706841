// Common device-side types for the sbt200 kernels (sm_100a).
//
// Every kernel computes the fully strided batched GEMM of the reference seam
// (reference _loops_numba.py:12-35):
//   C[i*crs + j*ccs + p*cps + q*cps2] = alpha * sum_l A[i*ars + l*acs + p*aps + q*aps2]
//                                              * B[l*brs + j*bcs + p*bps + q*bps2]
//                                     + beta * C[...]
// with base pointers already offset by (oa, ob, oc).  q is the optional second
// batch mode that fuses the planner's LoopStep (planner.py:551-581).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sbt {

template <typename T>
struct GemmParams {
  int64_t m, n, k, batch, batch2;
  const T* a;
  int64_t ars, acs, aps, aps2;
  const T* b;
  int64_t brs, bcs, bps, bps2;
  T* c;
  int64_t crs, ccs, cps, cps2;
  T alpha, beta;
};

// Host-side bookkeeping shared by every launcher (defined in sbt_api.cu).
void note_launch(const char* kernel_name);
// cudaFuncAttributeMaxDynamicSharedMemorySize for `fn` on the CURRENT device
// (cached per (kernel, device)); 0 or SBT_ECUDA with sbt_last_error set.
int set_smem_attr(const void* fn, int bytes);
// record a CUDA failure of a launcher for sbt_last_error(); returns SBT_ECUDA
int cuda_fail(cudaError_t e, const char* what);
int kernel_override();  // 0 auto, 1 generic, 2 tensor-core tiled, 3 small-matrix
int accumulation_mode();  // this thread's sbt_set_accumulation (1 unbiased, 0 fast)
constexpr int kNumSMs = 148;

__host__ __device__ constexpr int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Store one output element with the reference's beta rule: C is never read
// when beta == 0 (reference test_kernels.py:28-34).
template <typename T>
__device__ __forceinline__ void store_out(T* cp, T acc, T alpha, T beta) {
  if (beta == T(0)) {
    *cp = alpha * acc;
  } else {
    *cp = alpha * acc + beta * *cp;
  }
}

}  // namespace sbt
