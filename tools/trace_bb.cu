// Tile timeline of the batch-blocked CTA-pair kernel on exceptional case 6.4
// (C[m,n,p] = A[k,p] B[n,k,m], n = 256; built with -DSBT_TRACE): per tile of
// CTA 0, MMA accumulator acquire / last issue and the direct-store epilogue.
#include <cstdio>
#include <vector>
#include "../paper_1606_05696_b200/csrc/sbt_common.cuh"
namespace sbt { void note_launch(const char*) {} int kernel_override() { return 0; } int accumulation_mode() { return 1; } }
#include "../paper_1606_05696_b200/csrc/sbt_dispatch.cuh"
using namespace sbt;
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 256;
  const size_t nb = size_t(n) * n * n, na = size_t(n) * n;
  float *a, *b, *c;
  cudaMalloc(&a, na * 4); cudaMalloc(&b, nb * 4); cudaMalloc(&c, nb * 4);
  cudaMemset(a, 0, na * 4); cudaMemset(b, 0, nb * 4);
  GemmParams<float> p{};
  p.m = n; p.n = n; p.k = n; p.batch = n; p.batch2 = 1;
  p.a = b; p.ars = int64_t(n) * n; p.acs = n; p.aps = 1;       // tensor B[n,k,m]: batch n unit-stride
  p.b = a; p.brs = 1; p.bcs = n; p.bps = 0;                     // tensor A[k,p]
  p.c = c; p.crs = 1; p.ccs = int64_t(n) * n; p.cps = n;        // C[m,n,p]
  p.alpha = 1.f; p.beta = 0.f;
  for (int r = 0; r < 3; ++r) launch_gemm<float>(p, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); launch_gemm<float>(p, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("n=%d %.4f ms %.1f TF/s err=%s\n", n, ms, 2.0 * n * double(n) * n * n / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  long long mma[64][2], epi[2][64][4];
  cudaMemcpyFromSymbol(mma, tf32tma::g_trace_mma, sizeof(mma));
  cudaMemcpyFromSymbol(epi, tf32tma::g_trace_epi, sizeof(epi));
  const long long t0 = mma[0][0];
  printf("tile  mma_acq  mma_end | epi_begin  epi_dur  tmem_ld   rest\n");
  for (int t = 0; t < 10; ++t)
    printf("%4d %8lld %8lld | %9lld %8lld %8lld %6lld\n", t, mma[t][0] - t0, mma[t][1] - t0,
           epi[0][t][0] - t0, epi[0][t][1] - epi[0][t][0], epi[0][t][2], epi[0][t][3]);
  std::vector<long long> tr(8 * 4096);
  cudaMemcpyFromSymbol(tr.data(), tf32tma::g_trace, tr.size() * 8);
  const char* names[4] = {"tma_slot_free", "conv_raw_landed", "conv_done", "mma_full"};
  for (int row = 0; row < 4; ++row) {
    printf("rank0 %-16s", names[row]);
    for (int g = 16; g < 40; ++g) printf(" %lld", tr[row * 4096 + g] ? (tr[row * 4096 + g] - t0) : -1);
    printf("\n");
  }
  return 0;
}
