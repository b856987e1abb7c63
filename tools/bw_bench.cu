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

// pass-like: prologue (coefficients into smem), 4 FMAs per row, epilogue
// (block reduction + atomics); `occ_smem` dynamic smem limits occupancy
template <int U, bool PRO, bool EPI>
__global__ void k_passlike(const double* __restrict__ V, int64_t tile_stride, int rows, const double* coef,
                           double* out, unsigned long long* acc) {
  extern __shared__ double sm[];
  const double2* p = reinterpret_cast<const double2*>(V + blockIdx.x * tile_stride) + threadIdx.x;
  if (PRO) {
    for (int i = threadIdx.x; i < 2 * rows; i += blockDim.x) sm[i] = coef[i];
    __syncthreads();
  }
  double a0 = 0, a1 = 0, q0 = 0, q1 = 0, b0 = 0, b1 = 0;
  for (int i = 0; i < rows; i += U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u < rows ? __ldcs(p + (int64_t)(i + u) * 128) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i + u >= rows) break;
      const double l = PRO ? sm[i + u] : 0.5, bb = PRO ? sm[rows + i + u] : 0.25;
      a0 = fma(l, v[u].x, a0); a1 = fma(l, v[u].y, a1);
      q0 = fma(v[u].x, v[u].x, q0); q1 = fma(v[u].y, v[u].y, q1);
      b0 = fma(v[u].x, bb, b0); b1 = fma(v[u].y, bb, b1);
    }
  }
  double r = a0 + a1 + q0 + q1 + b0 + b1;
  if (EPI) {
    __shared__ double red[4];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r;
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(acc, (unsigned long long)(red[0] + red[1] + red[2] + red[3]));
  }
  if (r == 1.2345) out[0] = r;
}

template <int U, bool PRO, bool EPI>
void run_pass(const char* name, const double* V, int64_t tiles, int64_t stride, int rows, const double* coef,
              double* out, unsigned long long* acc, size_t occ_smem) {
  cudaFuncSetAttribute(k_passlike<U, PRO, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)occ_smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_passlike<U, PRO, EPI><<<(unsigned)tiles, 128, occ_smem>>>(V, stride, rows, coef, out, acc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double bytes = (double)tiles * rows * 256 * 8;
  printf("%-34s %.1f us  %.0f GB/s  (%s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}


// ---- TMA bulk-copy stream: persistent CTAs, STAGES-deep ring of RPS rows
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(smem_addr(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}

template <int STAGES, int RPS>
__global__ void __launch_bounds__(160) k_tma_stream(const double* __restrict__ V, int64_t tile_stride, int rows,
                                                    int tiles, double* out, unsigned long long* acc) {
  extern __shared__ __align__(128) double ring[];  // [STAGES][RPS][256]
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x;
  const int chunks = (rows + RPS - 1) / RPS;
  const int my_tiles = tiles > (int)blockIdx.x ? (tiles - 1 - (int)blockIdx.x) / gridDim.x + 1 : 0;
  const int total = my_tiles * chunks;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= 128) {  // producer warp
    if (tid == 128) {
      for (int it = 0; it < total; ++it) {
        const int slot = it % STAGES, round = it / STAGES;
        if (round > 0) mbar_wait(&empty[slot], (round - 1) & 1);
        const int t = blockIdx.x + (it / chunks) * gridDim.x, c = it % chunks;
        const int r0 = c * RPS, nr = min(RPS, rows - r0);
        const uint32_t bytes = (uint32_t)nr * 256 * 8;
        mbar_expect_tx(&full[slot], bytes);
        bulk_copy(ring + (size_t)slot * RPS * 256, V + (int64_t)t * tile_stride + (int64_t)r0 * 256, bytes, &full[slot]);
      }
    }
    return;
  }
  double a0 = 0, a1 = 0, q0 = 0, q1 = 0, b0 = 0, b1 = 0, tot = 0;
  for (int it = 0; it < total; ++it) {
    const int slot = it % STAGES, round = it / STAGES;
    const int c = it % chunks, r0 = c * RPS, nr = min(RPS, rows - r0);
    mbar_wait(&full[slot], round & 1);
    const double2* src = reinterpret_cast<const double2*>(ring + (size_t)slot * RPS * 256) + tid;
#pragma unroll
    for (int r = 0; r < RPS; ++r) {
      if (r < nr) {
        const double2 v = src[r * 128];
        const double l = 0.5, bb = 0.25;
        a0 = fma(l, v.x, a0); a1 = fma(l, v.y, a1);
        q0 = fma(v.x, v.x, q0); q1 = fma(v.y, v.y, q1);
        b0 = fma(v.x, bb, b0); b1 = fma(v.y, bb, b1);
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[slot]);
    if (c == chunks - 1) {  // tile epilogue (reduction)
      tot += a0 + a1 + q0 + q1 + b0 + b1;
      a0 = a1 = q0 = q1 = b0 = b1 = 0;
    }
  }
  if (tot == 1.2345) out[0] = tot;
}

template <int STAGES, int RPS>
void run_tma(const char* name, const double* V, int64_t tiles, int64_t stride, int rows, double* out,
             unsigned long long* acc, int ctas_per_sm) {
  const size_t smem = (size_t)STAGES * RPS * 256 * 8;
  cudaFuncSetAttribute(k_tma_stream<STAGES, RPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  const int grid = 148 * ctas_per_sm;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_tma_stream<STAGES, RPS><<<grid, 160, smem>>>(V, stride, rows, (int)tiles, out, acc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double bytes = (double)tiles * rows * 256 * 8;
  printf("%-34s %.1f us  %.0f GB/s  (%s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
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
  double* coef;
  unsigned long long* acc;
  cudaMalloc(&coef, 8 * 1024); cudaMemset(coef, 0, 8 * 1024);
  cudaMalloc(&acc, 8);
  run_pass<4, false, false>("pass-like bare, 16 CTA/SM", V, tiles, stride, rows, coef, out, acc, 4096);
  run_pass<4, false, false>("pass-like bare, 10 CTA/SM", V, tiles, stride, rows, coef, out, acc, 21 * 1024);
  run_pass<4, true, false>("pass-like +prologue, 10 CTA/SM", V, tiles, stride, rows, coef, out, acc, 21 * 1024);
  run_pass<4, true, true>("pass-like +pro+epi, 10 CTA/SM", V, tiles, stride, rows, coef, out, acc, 21 * 1024);
  run_pass<4, true, true>("pass-like +pro+epi, 16 CTA/SM", V, tiles, stride, rows, coef, out, acc, 4096);
  run_pass<8, true, true>("pass-like U8 +pro+epi, 16 CTA/SM", V, tiles, stride, rows, coef, out, acc, 4096);
  run_tma<6, 8>("tma 6x16KB, 2 CTA/SM", V, tiles, stride, rows, out, acc, 2);
  run_tma<4, 8>("tma 4x16KB, 3 CTA/SM", V, tiles, stride, rows, out, acc, 3);
  run_tma<12, 4>("tma 12x8KB, 2 CTA/SM", V, tiles, stride, rows, out, acc, 2);
  run_tma<3, 16>("tma 3x32KB, 2 CTA/SM", V, tiles, stride, rows, out, acc, 2);
  run_tma<8, 8>("tma 8x16KB, 1 CTA/SM", V, tiles, stride, rows, out, acc, 1);
  return 0;
}
