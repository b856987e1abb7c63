// Diagnostic: is FP64 mma.sync m8n8k4 (DMMA) bit-identical to an ascending
// chain of fused multiply-adds d = fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c))))?
// If so, a blocked forward solve built from chained DMMAs reproduces the
// FMA-chain arithmetic of the streaming rebuild bit for bit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_order tools/dmma_order.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

__global__ void k_dmma(const double* A, const double* B, const double* C, double* D, double* F, int chains) {
  // one warp per trial: A 8x4 (row), B 4x8 (col), C 8x8; `chains` k-steps chained
  const int lane = threadIdx.x & 31;
  const int trial = blockIdx.x;
  const double* a = A + (size_t)trial * chains * 32;
  const double* b = B + (size_t)trial * chains * 32;
  const double* c = C + (size_t)trial * 64;
  // fragment layout (PTX ISA, mma.m8n8k4 .f64): A: row = lane/4, k = lane%4;
  // B: k = lane%4, col = lane/4; C/D: row = lane/4, cols 2*(lane%4) + {0,1}
  const int r = lane >> 2, q = lane & 3;
  double d0 = c[r * 8 + 2 * q], d1 = c[r * 8 + 2 * q + 1];
  for (int s = 0; s < chains; ++s) {
    const double av = a[s * 32 + r * 4 + q];
    const double bv = b[s * 32 + q * 8 + r];
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(av), "d"(bv));
  }
  D[(size_t)trial * 64 + r * 8 + 2 * q] = d0;
  D[(size_t)trial * 64 + r * 8 + 2 * q + 1] = d1;
  // reference: ascending FMA chain per element
  for (int e = lane; e < 64; e += 32) {
    const int i = e / 8, j = e % 8;
    double acc = c[e];
    for (int s = 0; s < chains; ++s)
      for (int k = 0; k < 4; ++k) acc = fma(a[s * 32 + i * 4 + k], b[s * 32 + k * 8 + j], acc);
    F[(size_t)trial * 64 + e] = acc;
  }
}

int main() {
  const int trials = 4096, chains = 55;
  std::mt19937_64 g(7);
  std::normal_distribution<double> nd;
  std::vector<double> A((size_t)trials * chains * 32), B(A.size()), C((size_t)trials * 64);
  for (auto& x : A) x = nd(g);
  for (auto& x : B) x = nd(g) * std::exp(nd(g));
  for (auto& x : C) x = nd(g);
  double *dA, *dB, *dC, *dD, *dF;
  cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dB, B.size() * 8); cudaMalloc(&dC, C.size() * 8);
  cudaMalloc(&dD, C.size() * 8); cudaMalloc(&dF, C.size() * 8);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice);
  k_dmma<<<trials, 32>>>(dA, dB, dC, dD, dF, chains);
  std::vector<double> D(C.size()), F(C.size());
  cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(F.data(), dF, F.size() * 8, cudaMemcpyDeviceToHost);
  size_t diff = 0;
  double worst = 0.0;
  for (size_t i = 0; i < D.size(); ++i)
    if (std::memcmp(&D[i], &F[i], 8)) {
      ++diff;
      worst = std::fmax(worst, std::fabs(D[i] - F[i]) / std::fmax(std::fabs(F[i]), 1e-300));
    }
  std::printf("{\"elements\": %zu, \"bit_different\": %zu, \"worst_rel\": %.3e, \"err\": \"%s\"}\n", D.size(), diff,
              worst, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
