// FP64 peak microbenchmarks on this GPU (SURVEY.md §8d asks for measured DFMA / DMMA peaks):
//   dfma: independent fused multiply-add chains on the FP64 pipe;
//   dmma: mma.sync.aligned.m8n8k4.row.col.f64 (the instruction k_schur_syrk uses).
// Prints one JSON line.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void k_dmma(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) dmma(acc[t][0], acc[t][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  // DFMA: blocks*threads*iters*16*8 FMAs, 2 flops each
  const int it_f = 4096;
  k_dfma<<<blocks, threads>>>(out, 16, 0.999, 1e-3);
  cudaEventRecord(e0);
  k_dfma<<<blocks, threads>>>(out, it_f, 0.999, 1e-3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms_f = 0;
  cudaEventElapsedTime(&ms_f, e0, e1);
  const double fl_f = 2.0 * blocks * threads * double(it_f) * 16 * 8;
  // DMMA: per warp iters*8 mma of 8x8x4 = 256 FMAs = 512 flops
  const int it_m = 8192;
  k_dmma<<<blocks, threads>>>(out, 16);
  cudaEventRecord(e0);
  k_dmma<<<blocks, threads>>>(out, it_m);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms_m = 0;
  cudaEventElapsedTime(&ms_m, e0, e1);
  const double fl_m = 512.0 * (blocks * threads / 32) * double(it_m) * 8;
  std::printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"sms\": %d, \"clock_khz\": %d, \"dfma_ms\": %.3f, "
              "\"dmma_ms\": %.3f, \"err\": \"%s\"}\n",
              fl_f / (ms_f * 1e-3) / 1e12, fl_m / (ms_m * 1e-3) / 1e12, sms, clk, ms_f, ms_m,
              cudaGetErrorString(cudaGetLastError()));
  return 0;
}
