// How many warps / independent chains does DMMA.8x8x4 need to saturate the fp64 pipe?
#include <cstdio>
template <int CH>
__global__ void k(double* out, int iters) {
  double acc[CH][2];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}
template <int CH>
void run(int warps_per_sm) {
  double* out; cudaMalloc(&out, 8);
  int threads = warps_per_sm * 32 > 1024 ? 1024 : warps_per_sm * 32;
  int blocks = 148 * (warps_per_sm * 32 / threads);
  int iters = 20000 / CH * 8;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<CH><<<blocks, threads>>>(out, 100);
  cudaEventRecord(e0); k<CH><<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * CH * double(iters) * blocks * threads / 32;
  printf("warps/SM %3d chains %2d: %.2f TFLOP/s\n", warps_per_sm, CH, fl / ms / 1e9);
}
int main() {
  for (int w : {4, 8, 16, 32}) { run<4>(w); run<8>(w); run<16>(w); run<32>(w); }
}
