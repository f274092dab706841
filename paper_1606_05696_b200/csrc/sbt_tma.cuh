// Host-side TMA tensor-map construction for strided GEMM operands.
//
// An operand view is (contiguous mode, other mode, batch, batch2) with element
// strides (1, s1, sb, sb2).  cuTensorMapEncodeTiled is fetched from the driver
// through cudaGetDriverEntryPoint (no link-time libcuda dependency).  Batch
// modes with stride 0 (broadcast operands) become extent-1 modes addressed at
// coordinate 0; out-of-range boxes are zero-filled by the TMA unit, which
// handles every M/N/K tail.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>

namespace sbt {

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 4-D fp32 view: dims (d0 contiguous, d1, batch, batch2), element strides
// (s1, sb, sb2), box (b0, b1, b2, 1).  Returns false if TMA cannot express it.
inline bool make_tmap_f32(CUtensorMap* map, const float* base, int64_t d0, int64_t d1,
                          int64_t s1, int64_t batch, int64_t sb, int64_t batch2, int64_t sb2,
                          uint32_t b0, uint32_t b1, CUtensorMapSwizzle swz, uint32_t b2 = 1) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[4] = {cuuint64_t(d0), cuuint64_t(d1), cuuint64_t(sb ? batch : 1),
                        cuuint64_t(sb2 ? batch2 : 1)};
  cuuint64_t strides[3] = {cuuint64_t(s1) * 4, cuuint64_t(sb ? sb : 4) * 4,
                           cuuint64_t(sb2 ? sb2 : 4) * 4};
  for (int i = 0; i < 3; ++i)
    if ((strides[i] & 15) || strides[i] >= (cuuint64_t(1) << 40)) return false;
  for (int i = 0; i < 4; ++i)
    if (dims[i] == 0 || dims[i] > (cuuint64_t(1) << 32)) return false;
  cuuint32_t box[4] = {b0, b1, b2, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  static const CUtensorMapL2promotion promo = [] {
    const char* v = std::getenv("SBT_TMA_L2PROMO");  // diagnostics: 0 none, 1 64B, 2 128B, 3 256B
    const int i = v ? std::atoi(v) : 3;
    return i == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
         : i == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : i == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                  : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, promo,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3-D fp64 view for the batched small-matrix DMMA kernel: dims (d0 contiguous,
// d1, batch) with element strides (s1, sb), box (b0, b1, b2).  b0 may exceed
// d0: the TMA zero-fills the extra rows, which pads the smem leading dimension.
inline bool make_tmap_f64_3d(CUtensorMap* map, const double* base, int64_t d0, int64_t d1,
                             int64_t s1, int64_t batch, int64_t sb, uint32_t b0, uint32_t b1,
                             uint32_t b2) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {cuuint64_t(d0), cuuint64_t(d1), cuuint64_t(batch)};
  cuuint64_t strides[2] = {cuuint64_t(s1) * 8, cuuint64_t(sb) * 8};
  for (int i = 0; i < 2; ++i)
    if ((strides[i] & 15) || strides[i] == 0 || strides[i] >= (cuuint64_t(1) << 40)) return false;
  if (b0 > 256 || b1 > 256 || b2 > 256) return false;
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace sbt
