// FP64 throughput microbenchmarks used as the roofline denominator
// (MEASURED_PEAKS.json carries no FP64 figure): a DMMA.8x8x4 loop and a DFMA
// loop over every SM, timed with CUDA events by the caller.
#include "kafmm_internal.h"

namespace kafmm {

__global__ void __launch_bounds__(256) k_peak_dmma(int iters, double* out) {
  double c[8][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 42.0) out[0] = s;
}

__global__ void __launch_bounds__(256) k_peak_dfma(int iters, double* out) {
  double c[8];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 42.0) out[0] = s;
}

}  // namespace kafmm

using namespace kafmm;

extern "C" kafmm_status kafmm_fp64_peak(int which, double* tflops) {
  if (!tflops) return KAFMM_EINVAL;
  try {
    int dev = 0, sms = 0;
    KF_CUDA(cudaGetDevice(&dev));
    KF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* d;
    KF_CUDA(cudaMalloc(&d, 8));
    cudaEvent_t e0, e1;
    KF_CUDA(cudaEventCreate(&e0));
    KF_CUDA(cudaEventCreate(&e1));
    const int blocks = sms * 4, threads = 256, iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {  // warm-up, then timed
      KF_CUDA(cudaEventRecord(e0));
      if (which == 0) k_peak_dmma<<<blocks, threads>>>(iters, d);
      else k_peak_dfma<<<blocks, threads>>>(iters, d);
      KF_CUDA(cudaEventRecord(e1));
      KF_CUDA(cudaEventSynchronize(e1));
    }
    float ms = 0;
    KF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    double flops = which == 0 ? (double)blocks * (threads / 32) * iters * 8 * 512.0  // 8x8x4 MACs x 2 per warp-op
                              : (double)blocks * threads * iters * 8 * 2.0;
    *tflops = flops / (ms * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return KAFMM_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.st;
  }
}
