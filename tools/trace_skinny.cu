// Timeline of the CTA-pair kernel on a skinny product (x0 = T x_0 U^T shape):
// C^T[(bc), z] = T^T[(bc), a] U[a, z], M' = 262144, N = 32, K = 512, K-major A and B.
#include <cstdio>
#include <vector>
#include "../paper_1606_05696_b200/csrc/sbt_common.cuh"
namespace sbt { void note_launch(const char* n) { printf("kernel %s\n", n); } int kernel_override() { return 0; } }
#include "../paper_1606_05696_b200/csrc/sbt_dispatch.cuh"
using namespace sbt;
int main(int argc, char** argv) {
  int64_t M = argc > 1 ? atol(argv[1]) : 262144, N = argc > 2 ? atol(argv[2]) : 32,
          K = argc > 3 ? atol(argv[3]) : 512;
  float *a, *b, *c;
  cudaMalloc(&a, M * K * 4); cudaMalloc(&b, K * N * 4); cudaMalloc(&c, M * N * 4);
  cudaMemset(a, 0, M * K * 4); cudaMemset(b, 0, K * N * 4);
  GemmParams<float> p{};
  p.m = M; p.n = N; p.k = K; p.batch = 1; p.batch2 = 1;
  p.a = a; p.ars = K; p.acs = 1;          // K-major A
  p.b = b; p.brs = 1; p.bcs = K;          // K-major B
  p.c = c; p.crs = N; p.ccs = 1;          // columns contiguous (as x0's C^T)
  p.alpha = 1.f; p.beta = 0.f;
  for (int r = 0; r < 3; ++r) launch_gemm<float>(p, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); launch_gemm<float>(p, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("M=%ld N=%ld K=%ld %.4f ms %.1f TF/s %.0f GB/s err=%s\n", M, N, K, ms, 2.0 * M * N * K / ms / 1e9,
         (M * K + K * N + M * N) * 4.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  std::vector<long long> tr(8 * 4096);
  cudaMemcpyFromSymbol(tr.data(), tf32tma::g_trace, tr.size() * 8);
  const char* names[4] = {"tma_slot_free", "conv_raw_landed", "conv_done", "mma_full"};
  for (int rk = 0; rk < 2; ++rk)
    for (int row = (rk ? 3 : 0); row < 4; ++row) {
      printf("rank%d %-16s", rk, names[row]);
      long long t0 = tr[0];
      for (int g = 0; g < 40; ++g) printf(" %lld", tr[(row + 4 * rk) * 4096 + g] ? (tr[(row + 4 * rk) * 4096 + g] - t0) : -1);
      printf("\n");
    }
  return 0;
}
