// DFMA latency / throughput microbenchmark on one SM-filling grid:
// CH independent dependent chains per thread, W warps per CTA (1 CTA per SM).
// Prints cycles per DFMA per warp and the FP64-pipe fraction (2 cycles per warp DFMA per SMSP = 100%).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (double)(t1 - t0) * 1e-300;
  if (threadIdx.x == 0 && blockIdx.x == 0) reinterpret_cast<long long*>(out)[gridDim.x * blockDim.x] = t1 - t0;
}
template <int CH>
void run(int warps) {
  double* d;
  cudaMalloc(&d, (148 * 1024 + 8) * 8);
  const int iters = 2000;
  k<CH><<<148, warps * 32>>>(d, iters, 1.0000001, 1e-9);
  k<CH><<<148, warps * 32>>>(d, iters, 1.0000001, 1e-9);
  cudaDeviceSynchronize();
  long long cyc;
  cudaMemcpy(&cyc, d + 148 * warps * 32, 8, cudaMemcpyDeviceToHost);
  const double n = (double)iters * 8 * CH;             // DFMA per warp
  const double per_smsp = n * (warps / 4.0);           // warp-DFMA per SMSP
  printf("chains %2d warps/SM %2d: %.2f cycles per DFMA per warp, pipe %.1f%%\n", CH, warps, cyc / n,
         100.0 * per_smsp * 2.0 / cyc);
  cudaFree(d);
}
int main() {
  for (int w : {4, 8, 12, 16}) {
    run<1>(w); run<2>(w); run<3>(w); run<4>(w); run<6>(w); run<8>(w);
  }
  return 0;
}
