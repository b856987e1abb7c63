// Diagnostic: FP64 throughput of this GPU -- DFMA (CUDA cores) and DMMA
// (mma.sync.m8n8k4.f64, the FP64 tensor-core path) -- to decide whether the
// dense triangular-solve contraction of the V rebuild belongs on DMMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = a + threadIdx.x + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

__global__ void k_dmma(double* out, double a, double b) {
  double fa = a + threadIdx.x, fb = b - threadIdx.x;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(fa), "d"(fb));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    k_dfma<<<blocks, threads>>>(out, 1.0, 0.999);
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, 1.0, 0.999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * kIters * (double)blocks * threads;
    std::printf("{\"kernel\": \"dfma\", \"ms\": %.4f, \"tflops\": %.2f}\n", ms, flops / ms / 1e9);
    k_dmma<<<blocks, threads>>>(out, 1.0, 0.999);
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(out, 1.0, 0.999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    // one m8n8k4 per warp = 8*8*4*2 flops
    const double mflops = 512.0 * 4 * kIters * (double)blocks * (threads / 32);
    std::printf("{\"kernel\": \"dmma_m8n8k4\", \"ms\": %.4f, \"tflops\": %.2f}\n", ms, mflops / ms / 1e9);
  }
  std::printf("{\"sms\": %d, \"clock_khz\": %d, \"err\": \"%s\"}\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
