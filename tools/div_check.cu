// Diagnostic: is the FMA-corrected quotient
//   y = __drcp_rn(b); q0 = a * y; r = fma(-q0, b, a); q = fma(r, y, q0)
// bit-identical to __ddiv_rn(a, b)?  (Markstein's correction with a
// correctly rounded reciprocal.)  Random normal operands over wide exponent
// ranges and random bit patterns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/div_check tools/div_check.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void k_check(uint64_t seed, int mode, unsigned long long* bad, unsigned long long* tested, double* ex) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned long long nb = 0, nt = 0;
  for (int it = 0; it < 64; ++it) {
    const uint64_t h1 = mix(seed ^ (i * 64 + it)), h2 = mix(h1 + 17);
    double a, b;
    if (mode == 0) {  // the rebuild's ranges: kernel values / residuals over pivots
      a = (double)(int64_t)(h1 >> 11) * 0x1p-53 * 2.0 - 1.0;
      a = ldexp(a, (int)(h1 % 60) - 50);
      b = ldexp(1.0 + (double)(h2 >> 12) * 0x1p-52, (int)(h2 % 40) - 30);
    } else {  // random bit patterns (normal range, away from overflow/underflow)
      const uint64_t ea = 1023 + (int)((h1 >> 52) % 1200) - 600, eb = 1023 + (int)((h2 >> 52) % 1200) - 600;
      a = __longlong_as_double((long long)((h1 & 0x800fffffffffffffull) | (ea << 52)));
      b = __longlong_as_double((long long)((h2 & 0x000fffffffffffffull) | (eb << 52)));
    }
    const double ref = __ddiv_rn(a, b);
    const double y = __drcp_rn(b);
    const double q0 = __dmul_rn(a, y);
    const double r = fma(-q0, b, a);
    const double q = fma(r, y, q0);
    ++nt;
    if (__double_as_longlong(q) != __double_as_longlong(ref)) {
      ++nb;
      ex[0] = a;
      ex[1] = b;
    }
  }
  atomicAdd(bad, nb);
  atomicAdd(tested, nt);
}

int main() {
  unsigned long long *bad, *tested;
  double* ex;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&tested, 8);
  cudaMallocManaged(&ex, 16);
  for (int mode = 0; mode < 2; ++mode) {
    *bad = *tested = 0;
    for (int rep = 0; rep < 16; ++rep) k_check<<<65536, 256>>>(1234567ull * (rep + 1) + mode, mode, bad, tested, ex);
    cudaDeviceSynchronize();
    printf("{\"mode\": %d, \"tested\": %llu, \"mismatch\": %llu, \"example\": [%.17g, %.17g]}\n", mode, *tested, *bad,
           ex[0], ex[1]);
  }
  return 0;
}
