// Diagnostic: dependent-chain latencies of FP64 ops, shuffles and shared
// memory on this GPU (clock64 around 1024-long chains, one warp).
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int iters) {
  __shared__ double sm[64];
  double x = a + threadIdx.x, y = b;
  long long t0, t1;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __dadd_rn(x, y);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __dmul_rn(x, y);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, a);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  // SHFL chain (double)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (i + 1) & 31);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
  // substitution step: x = shfl(acc * r), acc = acc - l * x
  double acc = x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const double xi = __shfl_sync(0xffffffffu, __dmul_rn(acc, y), i & 31);
    acc = __dadd_rn(acc, -__dmul_rn(a, xi));
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // smem round trip chain
  sm[threadIdx.x] = x;
  __syncwarp();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    volatile double* v = sm;
    v[(threadIdx.x + 1) & 31] = x;
    __syncwarp();
    x = v[threadIdx.x];
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
  out[threadIdx.x] = x + acc;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 8 * 64); cudaMallocManaged(&c, 8 * 8);
  const int it = 1024;
  for (int rep = 0; rep < 2; ++rep) { k<<<1, 32>>>(o, c, 1.0000001, 0.9999999, it); cudaDeviceSynchronize(); }
  const char* names[] = {"dadd", "dmul", "dfma", "shfl", "subst-step", "smem-rt"};
  for (int i = 0; i < 6; ++i) printf("%-12s %.1f cyc/op\n", names[i], (double)c[i] / it);
  return 0;
}
