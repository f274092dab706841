// Tile timeline of the CTA-pair kernel on the 4th-order contraction
// C[m,n,p,q] = A[m,k,p] B[n,k,q] (n = 128: p folded into M, q into N), built
// with -DSBT_TRACE: per tile of CTA 0, when the MMA warp got an accumulator
// and finished issuing, and when the TMA-store epilogue waited / got it /
// released it / finished.  Usage: trace_order4 [n] [k]
#include <cstdio>
#include <vector>
#include "../paper_1606_05696_b200/csrc/sbt_common.cuh"
namespace sbt { void note_launch(const char*) {} int kernel_override() { return 0; } int accumulation_mode() { return 1; } }
#include "../paper_1606_05696_b200/csrc/sbt_dispatch.cuh"
using namespace sbt;
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 128, k = argc > 2 ? atoi(argv[2]) : 128;
  const size_t na = size_t(n) * k * n, nc = size_t(n) * n * n * n;
  float *a, *b, *c;
  cudaMalloc(&a, na * 4); cudaMalloc(&b, na * 4); cudaMalloc(&c, nc * 4);
  cudaMemset(a, 0, na * 4); cudaMemset(b, 0, na * 4);
  GemmParams<float> p{};
  p.m = n; p.n = n; p.k = k; p.batch = n; p.batch2 = n;
  p.a = a; p.ars = 1; p.acs = n; p.aps = int64_t(n) * k; p.aps2 = 0;
  p.b = b; p.brs = n; p.bcs = 1; p.bps = 0; p.bps2 = int64_t(n) * k;
  p.c = c; p.crs = 1; p.ccs = n; p.cps = int64_t(n) * n; p.cps2 = int64_t(n) * n * n;
  p.alpha = 1.f; p.beta = 0.f;
  for (int r = 0; r < 3; ++r) launch_gemm<float>(p, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); launch_gemm<float>(p, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("n=%d k=%d %.4f ms %.1f TF/s err=%s\n", n, k, ms, 2.0 * n * n * double(k) * n * n / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  long long mma[64][2], epi[2][64][8];
  cudaMemcpyFromSymbol(mma, tf32tma::g_trace_mma, sizeof(mma));
  cudaMemcpyFromSymbol(epi, tf32tma::g_trace_tepi, sizeof(epi));
  const long long t0 = mma[0][0];
  printf("tile  mma_acq  mma_end | epi_wait  epi_acq  epi_rel  epi_end | tmem+cvt  bulkwait  sts+bar\n");
  for (int t = 0; t < 12; ++t)
    printf("%4d %8lld %8lld | %8lld %8lld %8lld %8lld | %8lld %8lld %8lld\n", t, mma[t][0] - t0,
           mma[t][1] - t0, epi[0][t][0] - t0, epi[0][t][1] - t0, epi[0][t][2] - t0,
           epi[0][t][3] - t0, epi[0][t][4], epi[0][t][5], epi[0][t][6]);
  return 0;
}
