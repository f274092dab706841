// Standalone timeline probe for the CTA-pair kernel (built with -DSBT_TRACE).
#include <cstdio>
#include <vector>
#include "../paper_1606_05696_b200/csrc/sbt_common.cuh"
namespace sbt { void note_launch(const char*) {} int kernel_override() { return 0; } int accumulation_mode() { return 1; } }
#include "../paper_1606_05696_b200/csrc/sbt_dispatch.cuh"
using namespace sbt;
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 256, P = argc > 2 ? atoi(argv[2]) : 256;
  size_t na = size_t(n) * n * P;
  float *a, *b, *c;
  cudaMalloc(&a, na * 4); cudaMalloc(&b, na * 4); cudaMalloc(&c, na * 4);
  cudaMemset(a, 0, na * 4); cudaMemset(b, 0, na * 4);
  GemmParams<float> p{};
  p.m = n; p.n = n; p.k = n; p.batch = P; p.batch2 = 1;
  p.a = a; p.ars = 1; p.acs = n; p.aps = int64_t(n) * n;
  p.b = b; p.brs = 1; p.bcs = n; p.bps = int64_t(n) * n;
  p.c = c; p.crs = 1; p.ccs = n; p.cps = int64_t(n) * n;
  p.alpha = 1.f; p.beta = 0.f;
  for (int r = 0; r < 3; ++r) launch_gemm<float>(p, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); launch_gemm<float>(p, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("n=%d P=%d %.4f ms %.1f TF/s err=%s\n", n, P, ms, 2.0 * n * n * double(n) * P / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  std::vector<long long> tr(8 * 4096);
  cudaMemcpyFromSymbol(tr.data(), tf32tma::g_trace, tr.size() * 8);
  const char* names[4] = {"tma_slot_free", "conv_raw_landed", "conv_done", "mma_full"};
  for (int rk = 0; rk < 2; ++rk)
    for (int row = (rk ? 3 : 0); row < 4; ++row) {
      printf("rank%d %-16s", rk, names[row]);
      long long t0 = tr[(0) * 4096];
      for (int g = 40; g < 72; ++g) printf(" %lld", tr[(row + 4 * rk) * 4096 + g] ? (tr[(row + 4 * rk) * 4096 + g] - t0) : -1);
      printf("\n");
    }
  long long ep[2][64][4];
  cudaMemcpyFromSymbol(ep, tf32tma::g_trace_epi, sizeof(ep));
  for (int rk = 0; rk < 2; ++rk)
    for (int t = 0; t < 5; ++t)
      printf("rank%d tile%d epi begin %lld dur %lld  tmem_ld %lld  rest %lld\n", rk, t,
             ep[rk][t][0] - tr[0], ep[rk][t][1] - ep[rk][t][0], ep[rk][t][2], ep[rk][t][3]);
  return 0;
}
