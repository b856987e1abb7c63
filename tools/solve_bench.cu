// Diagnostic: the single-CTA forward solve (cta_forward_solve) alone, on a
// synthetic well-conditioned packed factor in shared memory, timed per phase
// with clock64.  Not part of the product.
#include "../paper_2111_14991_b200/csrc/gtc_kernels.cu"

#include <cstdio>
#include <vector>

__global__ void k_solve(const double* Lg, const double* bg, int n, double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* Ls = sm;
  const int64_t np = gtc::packed(n);
  double* x = Ls + ((np + 1) & ~1LL);
  double* rinv = x + n;
  for (int64_t i = threadIdx.x; i < np; i += blockDim.x) Ls[i] = Lg[i];
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = bg[i];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) rinv[i] = __drcp_rn(Ls[gtc::packed(i) + i]);
  __syncthreads();
  long long t0 = clock64();
  gtc::cta_forward_solve(Ls, n, x, rinv);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = x[i];
}

// variant of gtc::cta_forward_solve with phase switches and per-phase clocks
template <int MODE>  // bit0: skip chain, bit1: skip folds, bit2: skip barrier
__device__ void solve_var(const double* Lp, int n, double* x, const double* rinv, long long* cyc) {
  using namespace gtc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblk = (n + 31) / 32;
  double lrd[32];
  double lf[32];
  double xr = 0.0, ri = 0.0;
  long long tch = 0, tbar = 0, tfold = 0;
  auto load_diag = [&](int blk) {
    const int b0 = 32 * blk, r = b0 + lane;
    const bool live = r < n;
    const double* Lr = Lp + packed(live ? r : b0) + b0;
#pragma unroll
    for (int k = 0; k < 32; ++k) lrd[k] = (live && k < lane) ? Lr[k] : 0.0;
    ri = live ? rinv[r] : 0.0;
  };
  if (warp == 0) {
    load_diag(0);
    xr = lane < n ? x[lane] : 0.0;
  }
  for (int s = 0; s < nblk; ++s) {
    const int b0 = 32 * s, kmax = min(32, n - b0);
    const int wn = (s + 1) % kSolveWarps;
    if (warp == wn && s + 1 < nblk) {
      const int r = b0 + 32 + lane;
      const bool live = r < n;
      const double* Lr = Lp + packed(live ? r : b0) + b0;
#pragma unroll
      for (int k = 0; k < 32; ++k) lf[k] = (live && k < kmax) ? Lr[k] : 0.0;
      load_diag(s + 1);
    }
    long long c0 = clock64();
    if (!(MODE & 1) && warp == s % kSolveWarps) {
      // branch-free (a shuffle under a divergent guard costs a convergence
      // check per step); lanes past n carry ri = 0, coefficients 0
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const double xi = __shfl_sync(0xffffffffu, __dmul_rn(xr, ri), k);
        const double upd = __dadd_rn(xr, -__dmul_rn(lrd[k], xi));
        xr = lane == k ? xi : (lane > k ? upd : xr);
      }
      if (b0 + lane < n) x[b0 + lane] = xr;
    }
    long long c1 = clock64();
    if (!(MODE & 4)) __syncthreads();
    long long c2 = clock64();
    if (!(MODE & 2) && s + 1 < nblk) {
      if (warp == wn) {
        const int r = b0 + 32 + lane;
        xr = r < n ? x[r] : 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (k < kmax) xr = __dadd_rn(xr, -__dmul_rn(lf[k], x[b0 + k]));
      } else if (!(MODE & 8)) {
        // far rows on the warps that do not share a scheduler with the next
        // chain (warps wn and wn + 4 share one of the 4 SM sub-partitions)
        const int wo = (wn + kSolveWarps / 2) % kSolveWarps;
        if (warp != wo) {
          const int t = threadIdx.x - 32 * ((warp > wn) + (warp > wo));
          for (int r = b0 + 64 + t; r < n; r += kCtaThreads - 64) fold_block(Lp, x, r, b0, kmax);
        }
      }
    }
    long long c3 = clock64();
    if (warp == s % kSolveWarps && lane == 0) { tch += c1 - c0; }
    if (threadIdx.x == 0) tbar += c2 - c1;
    if (warp == wn && lane == 0) tfold += c3 - c2;
    if (lane == 0) { atomicAdd((unsigned long long*)&cyc[1], (unsigned long long)(warp == s % kSolveWarps ? c1 - c0 : 0)); }
  }
  __syncthreads();
  if (threadIdx.x == 0) { cyc[2] = tbar; }
  if (lane == 0) { atomicAdd((unsigned long long*)&cyc[3], (unsigned long long)tfold); }
}

template <int MODE>
__global__ void k_solve_var(const double* Lg, const double* bg, int n, double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* Ls = sm;
  const int64_t np = gtc::packed(n);
  double* x = Ls + ((np + 1) & ~1LL);
  double* rinv = x + n;
  for (int64_t i = threadIdx.x; i < np; i += blockDim.x) Ls[i] = Lg[i];
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = bg[i];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) rinv[i] = __drcp_rn(Ls[gtc::packed(i) + i]);
  __syncthreads();
  long long t0 = clock64();
  solve_var<MODE>(Ls, n, x, rinv, cyc);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = x[i];
}

int main() {
  const int n = 219;
  const int64_t np = (int64_t)n * (n + 1) / 2;
  std::vector<double> L(np), b(n);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < i; ++j) L[(int64_t)i * (i + 1) / 2 + j] = 0.01 * ((i * 7 + j * 13) % 17 - 8) / (1 + i);
    L[(int64_t)i * (i + 1) / 2 + i] = 1.0 + 0.001 * i;
    b[i] = 1.0 + 0.01 * (i % 5);
  }
  double *dL, *db, *dout;
  long long* cyc;
  cudaMalloc(&dL, 8 * np); cudaMalloc(&db, 8 * n); cudaMalloc(&dout, 8 * n); cudaMallocManaged(&cyc, 64);
  cudaMemcpy(dL, L.data(), 8 * np, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), 8 * n, cudaMemcpyHostToDevice);
  const size_t smem = 8 * (((np + 1) & ~1LL) + 2 * n);
  cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int r = 0; r < 3; ++r) {
    k_solve<<<1, gtc::kCtaThreads, smem>>>(dL, db, n, dout, cyc);
    cudaDeviceSynchronize();
  }
  // reference on the host in the same order
  std::vector<double> x(b);
  for (int i = 0; i < n; ++i) {
    double acc = x[i];
    for (int j = 0; j < i; ++j) acc = acc - L[(int64_t)i * (i + 1) / 2 + j] * x[j];
    x[i] = acc * (1.0 / L[(int64_t)i * (i + 1) / 2 + i]);
  }
  std::vector<double> got(n);
  k_solve<<<1, gtc::kCtaThreads, smem>>>(dL, db, n, dout, cyc);
  cudaDeviceSynchronize();
  cudaMemcpy(got.data(), dout, 8 * n, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < n; ++i) err = std::max(err, std::abs(got[i] - x[i]));
  auto runv = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int r = 0; r < 3; ++r) {
      memset(cyc, 0, 64);
      kern<<<1, gtc::kCtaThreads, smem>>>(dL, db, n, dout, cyc);
      cudaDeviceSynchronize();
    }
    printf("%-22s total %6lld  chain(sum) %6lld  barrier(t0) %6lld  fold(next-warp sum) %6lld\n", name, cyc[0], cyc[1], cyc[2], cyc[3]);
  };
  runv(k_solve_var<0>, "full");
  runv(k_solve_var<2>, "no folds");
  runv(k_solve_var<1>, "no chain");
  runv(k_solve_var<8>, "no far folds");
  runv(k_solve_var<3>, "no chain no folds");
  printf("n=%d solve %lld cycles (%.2f us @1.965GHz), max |diff| vs host %.3g, err=%s\n", n, cyc[0], cyc[0] / 1965.0,
         err, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
