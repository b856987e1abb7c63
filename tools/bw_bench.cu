// Diagnostic: read-bandwidth ceiling for the pass's access pattern (tile-major
// V, one CTA per 256-candidate tile, double2 per thread per row) and variants.
#include <cstdio>
#include <cstdint>

template <int U, int THREADS, int VEC>
__global__ void k_read(const double* __restrict__ V, int64_t tile_stride, int rows, double* out) {
  // VEC = doubles per thread per row (2 or 4); THREADS * VEC = 256 candidates per row
  const double* base = V + blockIdx.x * tile_stride;
  double acc = 0.0;
  if (VEC == 2) {
    const double2* p = reinterpret_cast<const double2*>(base) + threadIdx.x;
    for (int i = 0; i < rows; i += U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = i + u < rows ? __ldcs(p + (int64_t)(i + u) * 128) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < U; ++u) acc = fma(v[u].x, v[u].y, acc);
    }
  } else {
    const double4* p = reinterpret_cast<const double4*>(base) + threadIdx.x;
    int i = 0;
    for (; i + U <= rows; i += U) {
      double4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double2* q = reinterpret_cast<const double2*>(p + (int64_t)(i + u) * 64);
        const double2 a = __ldcs(q), b = __ldcs(q + 1);
        v[u] = make_double4(a.x, a.y, b.x, b.y);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc = fma(v[u].x, v[u].y, acc) + v[u].z * v[u].w;
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

template <int U, int THREADS, int VEC>
void run(const char* name, const double* V, int64_t tiles, int64_t stride, int rows, double* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_read<U, THREADS, VEC><<<(unsigned)tiles, THREADS>>>(V, stride, rows, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double bytes = (double)tiles * rows * 256 * 8;
  printf("%-28s %.1f us  %.0f GB/s  (%s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t tiles = 3907;
  const int rows = 219, nmax = 220;
  const int64_t stride = (int64_t)nmax * 256;
  double *V, *out;
  cudaMalloc(&V, sizeof(double) * tiles * stride);
  cudaMalloc(&out, 64);
  cudaMemset(V, 0, sizeof(double) * tiles * stride);
  run<2, 128, 2>("U2  128thr double2", V, tiles, stride, rows, out);
  run<4, 128, 2>("U4  128thr double2", V, tiles, stride, rows, out);
  run<6, 128, 2>("U6  128thr double2", V, tiles, stride, rows, out);
  run<8, 128, 2>("U8  128thr double2", V, tiles, stride, rows, out);
  run<12, 128, 2>("U12 128thr double2", V, tiles, stride, rows, out);
  run<16, 128, 2>("U16 128thr double2", V, tiles, stride, rows, out);
  return 0;
}
