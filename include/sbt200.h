/*
 * sbt200 -- C ABI of the B200 (sm_100a) extended-BLAS tensor-contraction library.
 *
 * This is the drop-in boundary for the reference's arithmetic seam
 * (reference: /root/reference/pkg/src/sbtensor/backend.py:29-31), i.e. the
 * functions every kernel entry point of kernels.py ends in.  At that seam the
 * reference has already lowered op flags to element strides, so every entry
 * point here is a fully strided (batched) GEMM over flat buffers:
 *
 *   C[oc + i*crs + j*ccs + p*cpt] = alpha * sum_l A[oa + i*ars + l*acs + p*apt]
 *                                           * B[ob + l*brs + j*bcs + p*bpt]
 *                                  + beta * C[...]         (C not read if beta == 0)
 *
 * Units: element (not byte) offsets and strides, int64, all >= 0 (a zero batch
 * stride broadcasts that operand, reference test_kernels.py:84-96).
 * Ownership: A and B are read, C is updated in place.  Device memory on the
 * device-pointer entry points: none for the contraction kernels themselves;
 * the split-K paths (few output tiles with a long reduction, e.g. Gram
 * matrices) draw a stream-ordered workspace from the device's default memory
 * pool (cudaMallocAsync / cudaFreeAsync, capturable in a CUDA graph; the pool
 * keeps released memory, so repeated calls of a shape do not allocate from the
 * driver).  A failed workspace allocation returns SBT_ECUDA with a message.
 * Errors: 0 on success, a negative SBT_E* code otherwise; sbt_last_error()
 * returns a message for the calling thread.  The reference cores do no
 * validation (validation lives in kernels.py); these entry points validate
 * extents, strides and pointers so a bad call can never fault the device.
 * Threading: re-entrant; work is enqueued on `stream` (a cudaStream_t, NULL =
 * legacy default stream) and is complete after a stream synchronise.  The
 * *_host variants take host buffers, copy in/out and synchronise before
 * returning (the numpy-buffer seam of the reference).
 */
#ifndef SBT200_H
#define SBT200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBT_OK 0
#define SBT_EINVAL (-1)       /* bad extent / stride / pointer */
#define SBT_EUNSUPPORTED (-2) /* no kernel for this request */
#define SBT_ECUDA (-3)        /* CUDA runtime error (message in sbt_last_error) */

/* Library version (major*10000 + minor*100 + patch). */
int sbt_version(void);
/* Message describing the last failure on the calling thread ("" if none). */
const char* sbt_last_error(void);
/* Number of device kernels this library has launched (process-wide). */
int64_t sbt_launch_count(void);
/* Name of the kernel family chosen for the most recent launch on this thread. */
const char* sbt_last_kernel(void);
/* Force a kernel family: 0 = auto, 1 = generic SIMT, 2 = tensor-core tiled,
   3 = small-matrix batched.  Used by tests to cover every path. */
int sbt_set_kernel_override(int which);
/* fp32 accumulation mode of the narrow (N <= 64) tensor-core tiles for the
   calling thread: 1 = unbiased (default: round-to-nearest TF32 split, step
   accumulators summed in round-to-nearest fp32), 0 = fast (the tensor core's
   truncating accumulator: a relative shrink of ~K/16 ulp, harmless where only
   directions matter, e.g. the HOOI factor-update products).  Returns the
   previous mode. */
int sbt_set_accumulation(int mode);

/* Diagnostics (not part of the reference seam): measured fp64 throughput in
   TFLOP/s of the DMMA tensor pipe (kind 0) or DFMA SIMT pipe (kind 1). */
int sbt_probe_fp64_peak(int kind, double* tflops);
/* Diagnostics: measured dense TF32 tensor-pipe throughput (tcgen05.mma
   kind::tf32, TFLOP/s); the 3xTF32 fp32 roofline is this / 3. */
int sbt_probe_tf32_peak(double* tflops);
/* The same probe run back to back for `seconds` (clocks under the power cap). */
int sbt_probe_tf32_sustained(double seconds, double* tflops);

/* ---- reference: tucker.py:63-76 leading_left_singular_vectors (the HOOI
        factor update).  Finishes one warm-started subspace sweep on the
        device: qz = [Q | Z] (2p rows of n doubles: the columns of Q, then of
        Z = G Q), m = [Q Z]^T Z (2p x p column-major) or NULL (Q^T Z is then
        formed in-kernel).  Writes the leading
        `rank` Ritz vectors, sign-fixed as tucker.py:71-75, to ut (rank rows of
        n) and, when yt is not NULL, Y = G U to yt (same shape, unsigned: the
        next sweep's basis), when ut32 is not NULL the sign-fixed vectors
        rounded to fp32 (same shape), their values (descending) to w, flag[0] = 1 when every residual
        ||G u - w u|| <= tol * w_max, rel[0] = max residual / w_max, rel[1] = the
        number of Jacobi sweeps, rel[2..4] phase cycle counts, rel[5] Newton refinement steps (6
        doubles).  One
        kernel, no host synchronisation; p <= 64. */
int sbt_ritz_f64(const double* qz, const double* m, int64_t n, int p, int rank, double tol,
                 double* ut, double* yt, float* ut32, double* w, int* flag, double* rel,
                 void* stream);

/* ---- reference: tucker.py:63-76 applied at tucker.py:160-167 (one warm
        HOOI factor update, device-finished).  y: a packed column-major
        tensor of `order` extents `dims` (fp32 or fp64 elements); n =
        dims[mode].  qt: the previous factor's p columns as rows of ldq
        doubles (p <= 64).  Forms Z = Y_(mode) Y_(mode)^T Q in fp64 straight
        from y (no unfolding copy; fp32 widened on load; deterministic) in the
        caller's workspace `ws` (sbt_hooi_factor_ws_bytes bytes, 16-byte
        aligned, no initialisation needed; one per stream), then
        finishes the sweep exactly as sbt_ritz_f64 with m = NULL.  Three
        launches, no host synchronisation, capturable. */
size_t sbt_hooi_factor_ws_bytes(int order, const int64_t* dims, int mode, int p);
int sbt_hooi_factor_f32(const float* y, int order, const int64_t* dims, int mode,
                        const double* qt, int64_t ldq, int p, int rank, double tol, void* ws,
                        size_t ws_bytes, double* ut, double* yt, float* ut32, double* w,
                        int* flag, double* rel, void* stream);
int sbt_hooi_factor_f64(const double* y, int order, const int64_t* dims, int mode,
                        const double* qt, int64_t ldq, int p, int rank, double tol, void* ws,
                        size_t ws_bytes, double* ut, double* yt, float* ut32, double* w,
                        int* flag, double* rel, void* stream);
/* ---- reference: tucker.py:87-123 (_mode_product_chain), one small product
        T x_mode U^T with fp64 accumulation: y packed (order, dims), U's p
        columns as rows of ldq doubles (p <= 64), out packed with extent p at
        `mode`.  Every output is an fp64 dot product over dims[mode] (fixed
        order) rounded once: the HOOI core product of fp32 tensors, whose norm
        the fit compares, carries no tensor-core accumulator truncation. */
int sbt_mode_product_acc64_f32(const float* y, int order, const int64_t* dims, int mode,
                               const double* qt, int64_t ldq, int p, float* out, void* stream);
int sbt_mode_product_acc64_f64(const double* y, int order, const int64_t* dims, int mode,
                               const double* qt, int64_t ldq, int p, double* out, void* stream);
/* ---- reference: tucker.py:164-168 (fit from ||G||).  out[0] = ||core||_2
        (fp64 sum of squares over `count` packed elements, fixed order),
        out[1 + f] = flags[f] for f < nflags (<= 64): the HOOI iteration's one
        device->host read. */
int sbt_hooi_status_f32(const float* core, int64_t count, const int* flags, int nflags,
                        double* out, void* stream);
int sbt_hooi_status_f64(const double* core, int64_t count, const int* flags, int nflags,
                        double* out, void* stream);

/* ---- reference: layout.py:202-215 permute_copy (the conventional strategy's
        explicit transposition, planner.py:620-713; NOT used by planned
        contractions).  dst is packed column-major; its mode i has extent
        dims[i] and is read from src with element stride src_strides[i]. */
int sbt_permute_f64(int order, const int64_t* dims, const double* src,
                    const int64_t* src_strides, double* dst, void* stream);
int sbt_permute_f32(int order, const int64_t* dims, const float* src,
                    const int64_t* src_strides, float* dst, void* stream);

/* ---- reference: _loops_numba.py:12-25 gemm_core (called by kernels.gemm, kernels.py:107) */
int sbt_gemm_core_f64(int64_t m, int64_t n, int64_t k, double alpha,
                      const double* a, int64_t oa, int64_t ars, int64_t acs,
                      const double* b, int64_t ob, int64_t brs, int64_t bcs,
                      double beta, double* c, int64_t oc, int64_t crs, int64_t ccs,
                      void* stream);
int sbt_gemm_core_f32(int64_t m, int64_t n, int64_t k, float alpha,
                      const float* a, int64_t oa, int64_t ars, int64_t acs,
                      const float* b, int64_t ob, int64_t brs, int64_t bcs,
                      float beta, float* c, int64_t oc, int64_t crs, int64_t ccs,
                      void* stream);

/* ---- reference: _loops_numba.py:28-35 batched_core (kernels.strided_batched_gemm,
        kernels.py:156-176 via _run_batched :245-266) */
int sbt_batched_core_f64(int64_t m, int64_t n, int64_t k, double alpha,
                         const double* a, int64_t oa, int64_t ars, int64_t acs, int64_t apt,
                         const double* b, int64_t ob, int64_t brs, int64_t bcs, int64_t bpt,
                         double beta, double* c, int64_t oc, int64_t crs, int64_t ccs,
                         int64_t cpt, int64_t batch, void* stream);
int sbt_batched_core_f32(int64_t m, int64_t n, int64_t k, float alpha,
                         const float* a, int64_t oa, int64_t ars, int64_t acs, int64_t apt,
                         const float* b, int64_t ob, int64_t brs, int64_t bcs, int64_t bpt,
                         float beta, float* c, int64_t oc, int64_t crs, int64_t ccs,
                         int64_t cpt, int64_t batch, void* stream);

/* ---- reference: _loops_numba.py:38-68 ext_batched_core (kernels.strided_batched_gemm_ex,
        kernels.py:207-225).  Same arithmetic; one operand has unit batch stride. */
int sbt_ext_batched_core_f64(int64_t m, int64_t n, int64_t k, double alpha,
                             const double* a, int64_t oa, int64_t ars, int64_t acs, int64_t apt,
                             const double* b, int64_t ob, int64_t brs, int64_t bcs, int64_t bpt,
                             double beta, double* c, int64_t oc, int64_t crs, int64_t ccs,
                             int64_t cpt, int64_t batch, void* stream);
int sbt_ext_batched_core_f32(int64_t m, int64_t n, int64_t k, float alpha,
                             const float* a, int64_t oa, int64_t ars, int64_t acs, int64_t apt,
                             const float* b, int64_t ob, int64_t brs, int64_t bcs, int64_t bpt,
                             float beta, float* c, int64_t oc, int64_t crs, int64_t ccs,
                             int64_t cpt, int64_t batch, void* stream);

/* ---- reference: planner.py:551-581 (LoopStep loop around one batched call).
        Two nested batch modes in ONE launch: index p in [0,batch) uses the
        *pt strides, q in [0,batch2) the *pt2 strides. */
int sbt_batched2_core_f64(int64_t m, int64_t n, int64_t k, double alpha,
                          const double* a, int64_t oa, int64_t ars, int64_t acs, int64_t apt,
                          int64_t apt2,
                          const double* b, int64_t ob, int64_t brs, int64_t bcs, int64_t bpt,
                          int64_t bpt2,
                          double beta, double* c, int64_t oc, int64_t crs, int64_t ccs,
                          int64_t cpt, int64_t cpt2, int64_t batch, int64_t batch2,
                          void* stream);
int sbt_batched2_core_f32(int64_t m, int64_t n, int64_t k, float alpha,
                          const float* a, int64_t oa, int64_t ars, int64_t acs, int64_t apt,
                          int64_t apt2,
                          const float* b, int64_t ob, int64_t brs, int64_t bcs, int64_t bpt,
                          int64_t bpt2,
                          float beta, float* c, int64_t oc, int64_t crs, int64_t ccs,
                          int64_t cpt, int64_t cpt2, int64_t batch, int64_t batch2,
                          void* stream);

/* ---- grouped execution (no reference counterpart: the reference runs its
        contractions one call at a time).  `count` INDEPENDENT strided batched
        GEMMs -- no problem's C may overlap another problem's A, B or C -- in
        as few launches as possible: problems the CTA-pair tcgen05 kernel takes
        share one persistent launch per kernel configuration (one pipeline
        fill / drain / tail instead of one per problem); the rest run as
        single calls.  Each descriptor has the batched2 entry point's meaning
        (alpha/beta are converted to the buffer type). */
typedef struct sbt_gemm_desc {
  int64_t m, n, k;
  double alpha, beta;
  const void* a; int64_t oa, ars, acs, apt, apt2;
  const void* b; int64_t ob, brs, bcs, bpt, bpt2;
  void* c; int64_t oc, crs, ccs, cpt, cpt2;
  int64_t batch, batch2;
} sbt_gemm_desc;
int sbt_batched_core_group_f32(int count, const sbt_gemm_desc* descs, void* stream);
int sbt_batched_core_group_f64(int count, const sbt_gemm_desc* descs, void* stream);

/* ---- host-buffer seam: the reference's cores take flat numpy buffers
        (backend.py:29-31).  These copy the touched span of A, B (and C) to the
        device, run the same kernels, copy C back and synchronise. */
int sbt_batched_core_host_f64(int64_t m, int64_t n, int64_t k, double alpha,
                              const double* a, int64_t oa, int64_t ars, int64_t acs, int64_t apt,
                              const double* b, int64_t ob, int64_t brs, int64_t bcs, int64_t bpt,
                              double beta, double* c, int64_t oc, int64_t crs, int64_t ccs,
                              int64_t cpt, int64_t batch);
int sbt_batched_core_host_f32(int64_t m, int64_t n, int64_t k, float alpha,
                              const float* a, int64_t oa, int64_t ars, int64_t acs, int64_t apt,
                              const float* b, int64_t ob, int64_t brs, int64_t bcs, int64_t bpt,
                              float beta, float* c, int64_t oc, int64_t crs, int64_t ccs,
                              int64_t cpt, int64_t batch);

#ifdef __cplusplus
}
#endif
#endif /* SBT200_H */
