// Diagnostic: dependent-chain latency (cycles per instruction) of FP64
// mma.sync m8n8k4 (DMMA) with 1, 2, 4 independent chains per warp, one warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_lat tools/dmma_lat.cu
#include <cstdio>
template <int C>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double d[C][2];
  for (int c = 0; c < C; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-3 + c;
  const double av = a + threadIdx.x, bv = b - threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(av), "d"(bv));
  }
  const long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < C; ++c) s += d[c][0] + d[c][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void kf(double* out, long long* cyc, double a, double b) {
  double x = threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) x = fma(x, a, b);
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; long long h;
  cudaMalloc(&o, 8 * 64); cudaMalloc(&c, 8);
  k<1><<<1, 32>>>(o, c, 1.0, 1e-9); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("dmma 1 chain: %.1f cycles/instr\n", h / 1024.0);
  k<2><<<1, 32>>>(o, c, 1.0, 1e-9); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("dmma 2 chains: %.1f cycles/step (2 instr)\n", h / 1024.0);
  k<4><<<1, 32>>>(o, c, 1.0, 1e-9); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("dmma 4 chains: %.1f cycles/step (4 instr)\n", h / 1024.0);
  k<8><<<1, 32>>>(o, c, 1.0, 1e-9); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("dmma 8 chains: %.1f cycles/step (8 instr)\n", h / 1024.0);
  kf<<<1, 32>>>(o, c, 1.0000001, 1e-9); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("dfma chain: %.1f cycles/instr\n", h / 1024.0);
  return 0;
}
