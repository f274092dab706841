// Kernel-family selection for one strided (batched) GEMM request.
//
// The reference picks its arithmetic core by entry point only
// (kernels.py:107,174,223).  Here the same request is routed by stride class:
//   K1/K2 tensor-core tiles  (aligned, unit-stride operands; TF32x3 / DMMA)
//   K3    small-matrix batched (n <= 64, many batch entries)
//   K4    generic SIMT       (anything else; always correct)
#pragma once
#include "sbt_common.cuh"
#include "k_generic.cuh"

namespace sbt {

template <typename T, int BM, int BN, int BK, int TM, int TN>
static void launch_generic_cfg(const GemmParams<T>& p, cudaStream_t stream, const char* name) {
  const int64_t tiles_m = ceil_div(p.m, BM), tiles_n = ceil_div(p.n, BN);
  const int64_t total = tiles_m * tiles_n * p.batch * p.batch2;
  const int64_t grid = total < int64_t(kNumSMs) * 32 ? total : int64_t(kNumSMs) * 32;
  const int a_m_fast = p.ars <= p.acs ? 1 : 0;
  const int b_k_fast = p.brs <= p.bcs ? 1 : 0;
  generic_gemm_kernel<T, BM, BN, BK, TM, TN>
      <<<dim3(unsigned(grid)), dim3(GenericCfg<T, BM, BN, BK, TM, TN>::NT), 0, stream>>>(
          p, tiles_m, tiles_n, total, a_m_fast, b_k_fast);
  note_launch(name);
}

template <typename T>
static void launch_generic(const GemmParams<T>& p, cudaStream_t stream) {
  const bool small = p.m <= 48 || p.n <= 48;
  if constexpr (sizeof(T) == 4) {
    if (small) launch_generic_cfg<T, 32, 32, 16, 2, 2>(p, stream, "generic_f32_32x32");
    else       launch_generic_cfg<T, 128, 128, 8, 8, 8>(p, stream, "generic_f32_128x128");
  } else {
    if (small) launch_generic_cfg<T, 32, 32, 8, 2, 2>(p, stream, "generic_f64_32x32");
    else       launch_generic_cfg<T, 64, 64, 8, 4, 4>(p, stream, "generic_f64_64x64");
  }
}

template <typename T>
static int launch_gemm(const GemmParams<T>& p, cudaStream_t stream) {
  launch_generic<T>(p, stream);
  return 0;
}

}  // namespace sbt
