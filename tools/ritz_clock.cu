// Per-phase cycle counts of the Jacobi steps in k_ritz.cuh (built with
// -DSBT_RITZ_CLOCK): rotation phase vs block-update phase.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "../paper_1606_05696_b200/csrc/k_ritz.cuh"
using namespace sbt;
int main() {
  const int n = 512;
  for (int p : {32, 48}) {
    // m = [Q Z]^T Z with H block = diag + small symmetric noise
    std::vector<double> m(2 * p * p, 0.0), qz(2 * p * n, 0.0);
    srand(1);
    for (int i = 0; i < p; ++i)
      for (int j = 0; j <= i; ++j) {
        double v = (i == j) ? 100.0 - i : 1e-3 * (rand() / double(RAND_MAX) - 0.5);
        m[i + j * 2 * p] = v;
        m[j + i * 2 * p] = v;
      }
    for (auto& x : qz) x = rand() / double(RAND_MAX);
    double *dm, *dq, *du, *dw, *drel;  // rel: 6 doubles
    int* df;
    cudaMalloc(&dm, m.size() * 8);
    cudaMalloc(&dq, qz.size() * 8);
    cudaMalloc(&du, p * n * 8);
    cudaMalloc(&dw, p * 8);
    cudaMalloc(&drel, 6 * 8);
    cudaMalloc(&df, 4);
    cudaMemcpy(dm, m.data(), m.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dq, qz.data(), qz.size() * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(ritz::ritz_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ritz::SMEM_BYTES);
    long long z[2] = {0, 0};
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpyToSymbol(ritz::g_ritz_clock, z, sizeof(z));
      ritz::ritz_kernel<<<ritz::kCluster, ritz::kThreads, ritz::SMEM_BYTES>>>(dq, dm, n, p, 32, 1e-7, du, nullptr, nullptr, dw, df, drel);
      cudaDeviceSynchronize();
    }
    long long c[2];
    double rel[5];
    cudaMemcpyFromSymbol(c, ritz::g_ritz_clock, sizeof(c));
    cudaMemcpy(rel, drel, sizeof(rel), cudaMemcpyDeviceToHost);
    const double steps = rel[1] * (p - 1);
    printf("p=%d sweeps=%.0f  -- %.0f  step %.0f cycles/step; phases %.0f %.0f %.0f  err=%s\n", p,
           rel[1], c[0] / steps, c[1] / steps, rel[2], rel[3], rel[4], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
