// sm_100a kernels of the BO surrogate pass.
//
// Reference algorithm (all citations /root/reference/proj/include/gridtune/):
//   Matern closed forms          gp.hpp:27-56
//   GpModel::fit (Gram, LLT, jitter escalation, standardisation)  gp.hpp:81-135
//   GpModel::predict / cross_covariance                           gp.hpp:150-193
//   mean posterior variance      strategies.hpp:394-397,406-407
//   contextual-variance lambda   acquisition.hpp:73-83, strategies.hpp:404-418
//   PI / EI / LCB                acquisition.hpp:12-42
//   best_candidate (masked argmax, lowest position on ties, first-candidate rule)
//                                portfolio.hpp:32-61
//
// Design: the reference refits the GP and re-solves the whole
// n x U triangular system every iteration.  Here V = L^-1 K* lives in HBM and
// each valid observation appends ONE row of L (single CTA, bordered Cholesky)
// and ONE row of V (k_extend<1>): per candidate, the new row is
//   v_n = (k(x_n, x*) - sum_{m<n} L_nm v_m) / L_nn
// which is exactly the last step of the reference's forward substitution, and
// the posterior mean/variance fall out of the same pass:
//   mu = sum_i v_i beta_i  (beta = L^-1 y_standardized),  var = max(s2 - sum_i v_i^2, 0).
// The pass streams V once (HBM-bound GEMV), so it is written for bandwidth:
// tile-major V, 16-byte streaming loads, 8 rows in flight per thread.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <atomic>
#include <cstdint>

#include "gtc_internal.h"

namespace gtc {

static std::atomic<uint64_t> g_launches{0};
uint64_t launches() { return g_launches.load(); }
static inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ------------------------------------------------------------ device helpers

template <int NU>
__device__ __forceinline__ double matern(double r, double lengthscale, double s2) {
  // gp.hpp:40-55 evaluation order: s = r / l; (s2 * poly(a)) * exp(-a)
  const double s = __ddiv_rn(r, lengthscale);
  if (NU == 0) return __dmul_rn(s2, exp(-s));
  if (NU == 1) {
    const double a = __dmul_rn(1.7320508075688772, s);
    return __dmul_rn(__dmul_rn(s2, __dadd_rn(1.0, a)), exp(-a));
  }
  const double a = __dmul_rn(2.2360679774997896, s);
  const double poly = __dadd_rn(__dadd_rn(1.0, a), __ddiv_rn(__dmul_rn(a, a), 3.0));
  return __dmul_rn(__dmul_rn(s2, poly), exp(-a));
}

__device__ __forceinline__ double matern_rt(int nu, double r, double lengthscale, double s2) {
  if (nu == 0) return matern<0>(r, lengthscale, s2);
  if (nu == 1) return matern<1>(r, lengthscale, s2);
  return matern<2>(r, lengthscale, s2);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed shuffle/smem tree).  All threads get the result.
__device__ double block_sum(double v, double* red /* >= 32 doubles smem */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = lane < nw ? red[lane] : 0.0;
  t = warp_sum(t);
  return t;
}

__device__ __forceinline__ bool visited_bit(const uint32_t* visited, int64_t j) {
  return (__ldg(visited + (j >> 5)) >> (j & 31)) & 1u;
}

// Solves L x = b in place (x in shared memory, length n) with one CTA, using
// the first n rows of the row-major lower factor L (ld = ldL).  32-row blocks:
// warp 0 substitutes the diagonal block with shuffles, then every thread
// applies the block to the trailing rows.  Per row the subtraction order is
// ascending column index, like the reference's forward substitution.
__device__ void cta_forward_solve(const double* L, int ldL, int n, double* x) {
  for (int b0 = 0; b0 < n; b0 += 32) {
    const int b1 = min(b0 + 32, n);
    if (threadIdx.x < 32) {
      const int r = b0 + threadIdx.x;
      double xr = r < b1 ? x[r] : 0.0;
      for (int i = b0; i < b1; ++i) {
        if (r == i) xr = __ddiv_rn(xr, L[(int64_t)i * ldL + i]);
        const double xi = __shfl_sync(0xffffffffu, xr, i - b0);
        if (r > i && r < b1) xr = __dadd_rn(xr, -__dmul_rn(L[(int64_t)r * ldL + i], xi));
      }
      if (r < b1) x[r] = xr;
    }
    __syncthreads();
    for (int r = b1 + threadIdx.x; r < n; r += blockDim.x) {
      double s = x[r];
      const double* Lr = L + (int64_t)r * ldL;
      for (int i = b0; i < b1; ++i) s = __dadd_rn(s, -__dmul_rn(Lr[i], x[i]));
      x[r] = s;
    }
    __syncthreads();
  }
}

// Standardisation + beta for the first n observations (gp.hpp:97-103,130).
// Sequential sums in thread 0 (n <= n_max, tiny) keep them order-stable.
__device__ void cta_stats_beta(const GpDev& g, int n) {
  __shared__ double s_mean, s_std;
  if (threadIdx.x == 0) {
    double mean = 0.0, stdv = 1.0;
    if (n > 0) {
      double sum = 0.0;
      for (int i = 0; i < n; ++i) sum = __dadd_rn(sum, g.y[i]);
      mean = __ddiv_rn(sum, (double)n);
      if (n > 1) {
        double ss = 0.0;
        for (int i = 0; i < n; ++i) {
          const double dv = __dadd_rn(g.y[i], -mean);
          ss = __dadd_rn(ss, __dmul_rn(dv, dv));
        }
        const double var = __ddiv_rn(ss, (double)n);
        stdv = var > 0.0 ? sqrt(var) : 1.0;
      }
    }
    s_mean = mean;
    s_std = stdv;
    g.sc->y_mean = mean;
    g.sc->y_std = stdv;
    g.sc->n = n;
  }
  __syncthreads();
  const double shift = __dadd_rn(s_mean, -g.sc->y0);
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    g.beta[i] = __ddiv_rn(__dadd_rn(g.c[i], -__dmul_rn(shift, g.e[i])), s_std);
  __syncthreads();
}

template <int NU>
__device__ double direct_kernel(const double* xa, const double* xb, int d, double l, double s2) {
  // (X.row(i) - X.row(j)).norm(), gp.hpp:110
  double ss = 0.0;
  for (int t = 0; t < d; ++t) {
    const double dv = __dadd_rn(xa[t], -xb[t]);
    ss = __dadd_rn(ss, __dmul_rn(dv, dv));
  }
  return matern<NU>(sqrt(ss), l, s2);
}

// Appends training point `row` (coords already in g.train_x[row]) to the
// factor: l = L^-1 g, pivot = k(0) + noise + jitter - |l|^2 (gp.hpp:105-121).
// Returns false (and records the failure) when the pivot is <= 0.
template <int NU>
__device__ bool cta_border_row(const GpDev& g, KernelParams k, double noise, double jitter,
                               int row, double* xs, double* red) {
  const double* xr = g.train_x + (int64_t)row * g.d;
  for (int m = threadIdx.x; m < row; m += blockDim.x)
    xs[m] = direct_kernel<NU>(g.train_x + (int64_t)m * g.d, xr, g.d, k.lengthscale, k.s2);
  __syncthreads();
  cta_forward_solve(g.L, g.n_max, row, xs);
  double part = 0.0;
  for (int m = threadIdx.x; m < row; m += blockDim.x) part = __dadd_rn(part, __dmul_rn(xs[m], xs[m]));
  const double sumsq = block_sum(part, red);
  const double diag = __dadd_rn(matern<NU>(0.0, k.lengthscale, k.s2), __dadd_rn(noise, jitter));
  const double x = __dadd_rn(diag, -sumsq);
  if (x <= 0.0) {  // Eigen LLT fails exactly when x <= 0 (a NaN pivot proceeds)
    if (threadIdx.x == 0) {
      g.sc->status = 1;
      g.sc->fail_row = row;
    }
    __syncthreads();
    return false;
  }
  double* Lrow = g.L + (int64_t)row * g.n_max;
  for (int m = threadIdx.x; m < row; m += blockDim.x) Lrow[m] = xs[m];
  if (threadIdx.x == 0) Lrow[row] = sqrt(x);
  __syncthreads();
  return true;
}

// c[row], e[row] from the new L row (prefix-stable forward substitution).
__device__ void cta_ce_row(const GpDev& g, int row, double* red) {
  const double* Lrow = g.L + (int64_t)row * g.n_max;
  double pc = 0.0, pe = 0.0;
  for (int m = threadIdx.x; m < row; m += blockDim.x) {
    pc = __dadd_rn(pc, __dmul_rn(Lrow[m], g.c[m]));
    pe = __dadd_rn(pe, __dmul_rn(Lrow[m], g.e[m]));
  }
  const double sc = block_sum(pc, red);
  const double se = block_sum(pe, red);
  if (threadIdx.x == 0) {
    const double yr = __dadd_rn(g.y[row], -g.sc->y0);
    g.c[row] = __ddiv_rn(__dadd_rn(yr, -sc), Lrow[row]);
    g.e[row] = __ddiv_rn(__dadd_rn(1.0, -se), Lrow[row]);
  }
  __syncthreads();
}

// ------------------------------------------------------------ GP kernels

template <int NU>
__global__ void __launch_bounds__(kCtaThreads) k_gp_factor(GpDev g, KernelParams k, double noise,
                                                           double jitter, int n) {
  extern __shared__ double xs[];
  __shared__ double red[32];
  if (threadIdx.x == 0) {
    g.sc->status = 0;
    g.sc->fail_row = -1;
    g.sc->jitter = jitter;
    g.sc->y0 = n > 0 ? g.y[0] : 0.0;
  }
  for (int row = threadIdx.x; row < n; row += blockDim.x) {  // squared norms (sequential in t)
    double s = 0.0;
    for (int t = 0; t < g.d; ++t) {
      const double v = g.train_x[(int64_t)row * g.d + t];
      s = __dadd_rn(s, __dmul_rn(v, v));
    }
    g.train_n2[row] = s;
  }
  __syncthreads();
  for (int row = 0; row < n; ++row) {
    if (!cta_border_row<NU>(g, k, noise, jitter, row, xs, red)) {
      if (threadIdx.x == 0) g.sc->n = 0;
      return;
    }
  }
  for (int row = 0; row < n; ++row) cta_ce_row(g, row, red);
  cta_stats_beta(g, n);
}

template <int NU>
__global__ void __launch_bounds__(kCtaThreads)
    k_gp_append(GpDev g, KernelParams k, double noise, SpaceDev sp, int64_t pos,
                const double* x_explicit, double y_new, int n0) {
  extern __shared__ double xs[];
  __shared__ double red[32];
  __shared__ double xnew[64];
  for (int t = threadIdx.x; t < g.d; t += blockDim.x) {
    const double v = pos >= 0 ? sp.coords[(int64_t)t * sp.n_pad + pos] : x_explicit[t];
    xnew[t] = v;
    g.train_x[(int64_t)n0 * g.d + t] = v;
  }
  if (threadIdx.x == 0) {
    g.y[n0] = y_new;
    g.sc->status = 0;
    g.sc->fail_row = -1;
    if (n0 == 0) g.sc->y0 = y_new;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int t = 0; t < g.d; ++t) s = __dadd_rn(s, __dmul_rn(xnew[t], xnew[t]));
    g.train_n2[n0] = s;
  }
  const double jitter = g.sc->jitter;
  if (!cta_border_row<NU>(g, k, noise, jitter, n0, xs, red)) return;
  cta_ce_row(g, n0, red);
  cta_stats_beta(g, n0 + 1);
}

__global__ void k_gp_truncate(GpDev g, int n) { cta_stats_beta(g, n); }

// ------------------------------------------------------------ V extension

struct ExtendArgs {
  SpaceDev sp;
  GpDev g;
  double* V;
  int64_t tile_stride;
  int n0, r, final_pass, check_status;
  double lengthscale, s2;
  double* mu;
  double* var;
};

// Rows [n0, n0+r) of V for every candidate, r <= R, streaming rows [0, n0)
// once.  One CTA per tile of kTile candidates, one double2 column pair per
// thread.  With final_pass the posterior mean/variance are produced too.
template <int R, int NU>
__global__ void __launch_bounds__(kExtendThreads) k_extend(ExtendArgs a) {
  if (a.check_status && a.g.sc->status != 0) return;  // bordered row failed: host refactors
  extern __shared__ double sm[];
  const int n0 = a.n0, r = a.r;
  const int ld = n0 + R;
  double* Ls = sm;             // [R][ld] coefficients of the new rows
  double* bs = sm + R * ld;    // [n0 + r] beta
  double* xn = bs + ld;        // [R][d] new training coords
  double* xn2 = xn + R * a.g.d;// [R] their squared norms
  for (int idx = threadIdx.x; idx < r * (n0 + r); idx += blockDim.x) {
    const int t = idx / (n0 + r), m = idx % (n0 + r);
    Ls[t * ld + m] = a.g.L[(int64_t)(n0 + t) * a.g.n_max + m];
  }
  if (a.final_pass)
    for (int m = threadIdx.x; m < n0 + r; m += blockDim.x) bs[m] = a.g.beta[m];
  for (int idx = threadIdx.x; idx < r * a.g.d; idx += blockDim.x)
    xn[idx] = a.g.train_x[(int64_t)n0 * a.g.d + idx];
  for (int t = threadIdx.x; t < r; t += blockDim.x) xn2[t] = a.g.train_n2[n0 + t];
  __syncthreads();

  const int64_t tile = blockIdx.x;
  const int64_t j0 = tile * kTile + 2 * threadIdx.x;
  const double2* Vt = reinterpret_cast<const double2*>(a.V + tile * a.tile_stride) + threadIdx.x;
  constexpr int kRowStride = kTile / 2;  // in double2

  double acc0[R], acc1[R];
#pragma unroll
  for (int t = 0; t < R; ++t) acc0[t] = acc1[t] = 0.0;
  double q0 = 0.0, q1 = 0.0, b0 = 0.0, b1 = 0.0;  // sum v^2, sum v*beta

  int i = 0;
  constexpr int U = (R == 1) ? 8 : 4;
  for (; i + U <= n0; i += U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(Vt + (int64_t)(i + u) * kRowStride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int t = 0; t < R; ++t) {
        if (t < r) {
          const double l = Ls[t * ld + i + u];
          acc0[t] = fma(l, v[u].x, acc0[t]);
          acc1[t] = fma(l, v[u].y, acc1[t]);
        }
      }
      if (a.final_pass) {
        const double bb = bs[i + u];
        q0 = fma(v[u].x, v[u].x, q0);
        q1 = fma(v[u].y, v[u].y, q1);
        b0 = fma(v[u].x, bb, b0);
        b1 = fma(v[u].y, bb, b1);
      }
    }
  }
  for (; i < n0; ++i) {
    const double2 v = __ldcs(Vt + (int64_t)i * kRowStride);
#pragma unroll
    for (int t = 0; t < R; ++t) {
      if (t < r) {
        const double l = Ls[t * ld + i];
        acc0[t] = fma(l, v.x, acc0[t]);
        acc1[t] = fma(l, v.y, acc1[t]);
      }
    }
    if (a.final_pass) {
      const double bb = bs[i];
      q0 = fma(v.x, v.x, q0);
      q1 = fma(v.y, v.y, q1);
      b0 = fma(v.x, bb, b0);
      b1 = fma(v.y, bb, b1);
    }
  }

  // candidate coordinates (SoA) and squared norms, gp.hpp:176-179 expansion
  const int d = a.sp.d;
  double c0n2 = 0.0, c1n2 = 0.0;
  for (int t = 0; t < d; ++t) {
    const double2 c = *reinterpret_cast<const double2*>(a.sp.coords + (int64_t)t * a.sp.n_pad + j0);
    c0n2 = __dadd_rn(c0n2, __dmul_rn(c.x, c.x));
    c1n2 = __dadd_rn(c1n2, __dmul_rn(c.y, c.y));
  }
  double vn0[R], vn1[R];
#pragma unroll
  for (int t = 0; t < R; ++t) {
    if (t < r) {
      double dot0 = 0.0, dot1 = 0.0;
      for (int s = 0; s < d; ++s) {
        const double2 c = *reinterpret_cast<const double2*>(a.sp.coords + (int64_t)s * a.sp.n_pad + j0);
        const double xv = xn[t * d + s];
        dot0 = __dadd_rn(dot0, __dmul_rn(xv, c.x));
        dot1 = __dadd_rn(dot1, __dmul_rn(xv, c.y));
      }
      // d2 = (-2 a.b + |a|^2) + |b|^2, clamp, sqrt  (gp.hpp:176-179)
      const double d20 = __dadd_rn(__dadd_rn(__dmul_rn(-2.0, dot0), xn2[t]), c0n2);
      const double d21 = __dadd_rn(__dadd_rn(__dmul_rn(-2.0, dot1), xn2[t]), c1n2);
      const double k0 = matern<NU>(sqrt(fmax(d20, 0.0)), a.lengthscale, a.s2);
      const double k1 = matern<NU>(sqrt(fmax(d21, 0.0)), a.lengthscale, a.s2);
      double num0 = __dadd_rn(k0, -acc0[t]);
      double num1 = __dadd_rn(k1, -acc1[t]);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        if (s < t) {
          const double l = Ls[t * ld + n0 + s];
          num0 = __dadd_rn(num0, -__dmul_rn(l, vn0[s]));
          num1 = __dadd_rn(num1, -__dmul_rn(l, vn1[s]));
        }
      }
      const double diag = Ls[t * ld + n0 + t];
      vn0[t] = __ddiv_rn(num0, diag);
      vn1[t] = __ddiv_rn(num1, diag);
      double2* dst = reinterpret_cast<double2*>(a.V + tile * a.tile_stride) + threadIdx.x +
                     (int64_t)(n0 + t) * kRowStride;
      *dst = make_double2(vn0[t], vn1[t]);
      if (a.final_pass) {
        const double bb = bs[n0 + t];
        q0 = fma(vn0[t], vn0[t], q0);
        q1 = fma(vn1[t], vn1[t], q1);
        b0 = fma(vn0[t], bb, b0);
        b1 = fma(vn1[t], bb, b1);
      }
    }
  }
  if (a.final_pass) {
    // mean = k*^T alpha = v^T beta;  var = max(s2 - sum v^2, 0)   (gp.hpp:162-166)
    *reinterpret_cast<double2*>(a.mu + j0) = make_double2(b0, b1);
    *reinterpret_cast<double2*>(a.var + j0) =
        make_double2(fmax(__dadd_rn(a.s2, -q0), 0.0), fmax(__dadd_rn(a.s2, -q1), 0.0));
  }
}

// Prior (n == 0): mean 0, variance = output variance (gp.hpp:155-158).
__global__ void k_prior(double* mu, double* var, int64_t n, double s2) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    mu[j] = 0.0;
    var[j] = s2;
  }
}

__global__ void k_mark(uint32_t* visited, int64_t pos, int set) {
  if (set)
    visited[pos >> 5] |= (1u << (pos & 31));
  else
    visited[pos >> 5] &= ~(1u << (pos & 31));
}

// ------------------------------------------------------------ reductions

int reduce_blocks(int64_t n) {
  const int64_t per_block = (int64_t)kReduceThreads * 8;
  int64_t b = (n + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > 148 * 8) b = 148 * 8;
  return (int)b;
}

// Last-block-done pattern: returns true in exactly one (the last) block.
__device__ bool last_block(unsigned int* counter) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  return is_last;
}

__global__ void __launch_bounds__(kReduceThreads)
    k_varsum(const double* __restrict__ var, const uint32_t* __restrict__ visited, int64_t n,
             double* partial_sum, int64_t* partial_cnt, unsigned int* counter, VarTotals* totals) {
  __shared__ double red[32];
  __shared__ unsigned long long cnt_s;
  if (threadIdx.x == 0) cnt_s = 0;
  __syncthreads();
  double s = 0.0;
  unsigned long long c = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (!visited_bit(visited, j)) {
      s += var[j];
      ++c;
    }
  }
  s = block_sum(s, red);
  atomicAdd(&cnt_s, c);
  __syncthreads();
  if (threadIdx.x == 0) {
    partial_sum[blockIdx.x] = s;
    partial_cnt[blockIdx.x] = (int64_t)cnt_s;
  }
  if (!last_block(counter)) return;
  double ts = 0.0;
  int64_t tc = 0;
  for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    ts += __ldcg(partial_sum + b);
    tc += __ldcg(reinterpret_cast<const long long*>(partial_cnt) + b);
  }
  ts = block_sum(ts, red);
  __shared__ unsigned long long tc_s;
  if (threadIdx.x == 0) tc_s = 0;
  __syncthreads();
  atomicAdd(&tc_s, (unsigned long long)tc);
  __syncthreads();
  if (threadIdx.x == 0) {
    totals->sum = ts;
    totals->count = (int64_t)tc_s;
    *counter = 0;
  }
}

// Acquisition functions, acquisition.hpp:12-42 (no FMA contraction).
__device__ __forceinline__ double normal_cdf(double z) {
  return __dmul_rn(0.5, erfc(__dmul_rn(-z, 0.70710678118654752440)));
}
__device__ __forceinline__ double normal_pdf(double z) {
  return __dmul_rn(0.3989422804014326779, exp(__dmul_rn(__dmul_rn(-0.5, z), z)));
}
__device__ __forceinline__ double acq_pi(double mean, double sd, double best, double lambda) {
  const double margin = __dadd_rn(__dadd_rn(best, lambda), -mean);
  if (sd <= 0.0) return margin > 0.0 ? 1.0 : 0.0;
  return normal_cdf(__ddiv_rn(margin, sd));
}
__device__ __forceinline__ double acq_ei(double mean, double sd, double best, double lambda) {
  const double margin = __dadd_rn(__dadd_rn(best, -lambda), -mean);
  if (sd <= 0.0) return margin > 0.0 ? margin : 0.0;
  const double z = __ddiv_rn(margin, sd);
  return __dadd_rn(__dmul_rn(margin, normal_cdf(z)), __dmul_rn(sd, normal_pdf(z)));
}
__device__ __forceinline__ double acq_neg_lcb(double mean, double sd, double lambda) {
  return -__dadd_rn(mean, -__dmul_rn(lambda, sd));
}
__device__ __forceinline__ double score_of(int af, double mean, double sd, double best, double lambda) {
  if (af == 0) return acq_ei(mean, sd, best, lambda);
  if (af == 1) return acq_pi(mean, sd, best, lambda);
  return acq_neg_lcb(mean, sd, lambda);
}

// (score, position) order used by best_candidate: higher score wins, lower
// position on ties; NaN scores never win (they are skipped, portfolio.hpp:52)
// except through the first-candidate rule applied at the end.
struct Best {
  double s;
  int64_t p;  // INT64_MAX = none
};
__device__ __forceinline__ Best better(Best a, Best b) {
  if (b.p == INT64_MAX) return a;
  if (a.p == INT64_MAX) return b;
  if (b.s > a.s || (b.s == a.s && b.p < a.p)) return b;
  return a;
}
__device__ __forceinline__ Best warp_best(Best v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Best w;
    w.s = __shfl_xor_sync(0xffffffffu, v.s, o);
    w.p = __shfl_xor_sync(0xffffffffu, v.p, o);
    v = better(v, w);
  }
  return v;
}
__device__ Best block_best(Best v, Best* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_best(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  Best t = lane < nw ? red[lane] : Best{0.0, INT64_MAX};
  return warp_best(t);
}
__device__ __forceinline__ int64_t warp_min(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, (int64_t)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ int64_t block_min(int64_t v, int64_t* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_min(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int64_t t = lane < nw ? red[lane] : INT64_MAX;
  return warp_min(t);
}

struct SelCtx {
  // scoring inputs
  const double* mu;
  const double* var;     // variance (run path) ...
  const double* sdv;     // ... or std (best_candidate path); exactly one is set
  const uint32_t* visited;
  const uint8_t* excluded_bytes;
  const int64_t* excluded_pos;
  int n_excluded;
  int64_t n;
  uint32_t af_mask;
  // partials
  double* partial_score;
  int64_t* partial_pos;
  int64_t* partial_first;
  int64_t* partial_cnt;
  unsigned int* counter;
  SelectDev* out;
};

__device__ __forceinline__ bool eligible(const SelCtx& c, int64_t j) {
  if (c.visited && visited_bit(c.visited, j)) return false;
  if (c.excluded_bytes && c.excluded_bytes[j]) return false;
  for (int k = 0; k < c.n_excluded; ++k)
    if (c.excluded_pos[k] == j) return false;
  return true;
}

__device__ __forceinline__ double sd_at(const SelCtx& c, int64_t j) {
  return c.sdv ? c.sdv[j] : sqrt(c.var[j]);  // cand_stds = sqrt(cand_vars), strategies.hpp:385
}

// Shared body of the selection: every block scans a strided slice, the last
// block merges.  lambda/best_std are provided by the caller (computed in the
// kernel prologue for the run path).
__device__ void select_body(const SelCtx& c, double best, double lambda, double mean_var,
                            int cv_fallback, int gp_status) {
  __shared__ Best redb[32];
  __shared__ int64_t redi[32];
  __shared__ unsigned long long cnt_s;
  if (threadIdx.x == 0) cnt_s = 0;
  __syncthreads();
  Best b[3] = {{0.0, INT64_MAX}, {0.0, INT64_MAX}, {0.0, INT64_MAX}};
  int64_t first = INT64_MAX;
  unsigned long long cnt = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < c.n;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (!eligible(c, j)) continue;
    ++cnt;
    first = min(first, j);
    const double m = c.mu[j], sd = sd_at(c, j);
#pragma unroll
    for (int af = 0; af < 3; ++af) {
      if (!(c.af_mask & (1u << af))) continue;
      const double s = score_of(af, m, sd, best, lambda);
      if (s == s) b[af] = better(b[af], Best{s, j});
    }
  }
  atomicAdd(&cnt_s, cnt);
  for (int af = 0; af < 3; ++af) b[af] = block_best(b[af], redb);
  first = block_min(first, redi);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int af = 0; af < 3; ++af) {
      c.partial_score[blockIdx.x * 3 + af] = b[af].s;
      c.partial_pos[blockIdx.x * 3 + af] = b[af].p;
    }
    c.partial_first[blockIdx.x] = first;
    c.partial_cnt[blockIdx.x] = (int64_t)cnt_s;
  }
  if (!last_block(c.counter)) return;
  Best f[3] = {{0.0, INT64_MAX}, {0.0, INT64_MAX}, {0.0, INT64_MAX}};
  int64_t ff = INT64_MAX;
  unsigned long long fc = 0;
  for (int blk = threadIdx.x; blk < gridDim.x; blk += blockDim.x) {
    for (int af = 0; af < 3; ++af)
      f[af] = better(f[af], Best{__ldcg(c.partial_score + blk * 3 + af),
                                 (int64_t)__ldcg(reinterpret_cast<const long long*>(c.partial_pos) + blk * 3 + af)});
    ff = min(ff, (int64_t)__ldcg(reinterpret_cast<const long long*>(c.partial_first) + blk));
    fc += (unsigned long long)__ldcg(reinterpret_cast<const long long*>(c.partial_cnt) + blk);
  }
  for (int af = 0; af < 3; ++af) f[af] = block_best(f[af], redb);
  ff = block_min(ff, redi);
  __shared__ unsigned long long fc_s;
  if (threadIdx.x == 0) fc_s = 0;
  __syncthreads();
  atomicAdd(&fc_s, fc);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int af = 0; af < 3; ++af) {
      int64_t pos = -1;
      double sc = 0.0;
      if ((c.af_mask & (1u << af)) && fc_s > 0) {
        // first-candidate rule (portfolio.hpp:52): the first eligible
        // candidate is taken unconditionally; if its score is NaN nothing
        // can beat it.
        const double s_first = score_of(af, c.mu[ff], sd_at(c, ff), best, lambda);
        if (s_first != s_first || f[af].p == INT64_MAX) {
          pos = ff;
          sc = s_first;
        } else {
          pos = f[af].p;
          sc = f[af].s;
        }
      }
      c.out->position[af] = pos;
      c.out->score[af] = sc;
    }
    c.out->lambda = lambda;
    c.out->mean_variance = mean_var;
    c.out->best_std = best;
    c.out->n_candidates = (int64_t)fc_s;
    c.out->cv_fallback = cv_fallback;
    c.out->gp_status = gp_status;
    *c.counter = 0;
  }
}

__global__ void __launch_bounds__(kReduceThreads)
    k_select(SelCtx c, const VarTotals* totals, const GpScalars* sc, SelectParams p) {
  // lambda (strategies.hpp:404-418, acquisition.hpp:73-83) and best_std
  // (gp.hpp:145), computed identically by every block.
  const double mean_var = totals->count > 0 ? __ddiv_rn(totals->sum, (double)totals->count) : 0.0;
  double lambda = p.lambda_constant;
  int fallback = 0;
  if (p.lambda_mode == 1) {
    if (!(p.f_best_raw > 0.0) || !(p.cv_mu_s > 0.0) || !(p.cv_var_s > 0.0)) {
      fallback = 1;
    } else {
      const double l = __ddiv_rn(__ddiv_rn(__dmul_rn(mean_var, p.f_best_raw), p.cv_mu_s), p.cv_var_s);
      lambda = l > 0.0 ? l : 0.0;
    }
  }
  const double best = __ddiv_rn(__dadd_rn(p.f_best_raw, -sc->y_mean), sc->y_std);
  select_body(c, best, lambda, mean_var, fallback, sc->status);
}

__global__ void __launch_bounds__(kReduceThreads)
    k_best_candidate(SelCtx c, double best, double lambda) {
  select_body(c, best, lambda, 0.0, 0, 0);
}

__global__ void k_scores(const double* __restrict__ mu, const double* __restrict__ sd, int64_t n,
                         int af, double best, double lambda, double* out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = score_of(af, mu[j], sd[j], best, lambda);
}

// ------------------------------------------------------------ launchers

static size_t cta_smem(int n_max) { return sizeof(double) * (size_t)(n_max + 8); }

void launch_gp_factor(const GpDev& g, KernelParams k, double noise, double jitter, int n,
                      cudaStream_t s) {
  count_launch();
  const size_t sm = cta_smem(g.n_max);
  switch (k.nu) {
    case 0: k_gp_factor<0><<<1, kCtaThreads, sm, s>>>(g, k, noise, jitter, n); break;
    case 1: k_gp_factor<1><<<1, kCtaThreads, sm, s>>>(g, k, noise, jitter, n); break;
    default: k_gp_factor<2><<<1, kCtaThreads, sm, s>>>(g, k, noise, jitter, n); break;
  }
}

void launch_gp_append(const GpDev& g, KernelParams k, double noise, const SpaceDev& sp,
                      int64_t pos, const double* x_explicit, double y_new, int n0, cudaStream_t s) {
  count_launch();
  const size_t sm = cta_smem(g.n_max);
  switch (k.nu) {
    case 0: k_gp_append<0><<<1, kCtaThreads, sm, s>>>(g, k, noise, sp, pos, x_explicit, y_new, n0); break;
    case 1: k_gp_append<1><<<1, kCtaThreads, sm, s>>>(g, k, noise, sp, pos, x_explicit, y_new, n0); break;
    default: k_gp_append<2><<<1, kCtaThreads, sm, s>>>(g, k, noise, sp, pos, x_explicit, y_new, n0); break;
  }
}

void launch_gp_truncate(const GpDev& g, int n, cudaStream_t s) {
  count_launch();
  k_gp_truncate<<<1, kCtaThreads, 0, s>>>(g, n);
}

template <int R, int NU>
static void extend_impl(const ExtendArgs& a, int64_t tiles, cudaStream_t s) {
  const size_t sm = sizeof(double) * ((size_t)(R + 1) * (a.n0 + R) + (size_t)R * a.g.d + R + 8);
  if (sm > 48 * 1024)  // rebuild passes at large n; set per call (per device context)
    cudaFuncSetAttribute(k_extend<R, NU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_extend<R, NU><<<(unsigned)tiles, kExtendThreads, sm, s>>>(a);
}

void launch_extend(const SpaceDev& sp, const GpDev& g, KernelParams k, double* V,
                   int64_t tile_stride, int n0, int r, bool final, double* mu, double* var,
                   bool check_status, cudaStream_t s) {
  count_launch();
  ExtendArgs a{sp, g, V, tile_stride, n0, r, final ? 1 : 0, check_status ? 1 : 0,
               k.lengthscale, k.s2, mu, var};
  const int64_t tiles = sp.n_pad / kTile;
  if (r == 1) {
    switch (k.nu) {
      case 0: extend_impl<1, 0>(a, tiles, s); break;
      case 1: extend_impl<1, 1>(a, tiles, s); break;
      default: extend_impl<1, 2>(a, tiles, s); break;
    }
  } else {
    switch (k.nu) {
      case 0: extend_impl<8, 0>(a, tiles, s); break;
      case 1: extend_impl<8, 1>(a, tiles, s); break;
      default: extend_impl<8, 2>(a, tiles, s); break;
    }
  }
}

void launch_prior(double* mu, double* var, int64_t n, double s2, cudaStream_t s) {
  count_launch();
  k_prior<<<148, 256, 0, s>>>(mu, var, n, s2);
}

void launch_mark(uint32_t* visited, int64_t pos, int set, cudaStream_t s) {
  count_launch();
  k_mark<<<1, 1, 0, s>>>(visited, pos, set);
}

void launch_varsum(const double* var, const uint32_t* visited, int64_t n, double* ps, int64_t* pc,
                   unsigned int* counter, VarTotals* totals, cudaStream_t s) {
  count_launch();
  k_varsum<<<reduce_blocks(n), kReduceThreads, 0, s>>>(var, visited, n, ps, pc, counter, totals);
}

void launch_select(const double* mu, const double* var, const uint32_t* visited, int64_t n,
                   const VarTotals* totals, const GpScalars* sc, SelectParams p,
                   double* partial_score, int64_t* partial_pos, int64_t* partial_first,
                   int64_t* partial_cnt, unsigned int* counter, SelectDev* out, cudaStream_t s) {
  count_launch();
  SelCtx c{mu, var, nullptr, visited, nullptr, p.excluded, p.n_excluded, n, p.af_mask,
           partial_score, partial_pos, partial_first, partial_cnt, counter, out};
  k_select<<<reduce_blocks(n), kReduceThreads, 0, s>>>(c, totals, sc, p);
}

void launch_best_candidate(const double* mu, const double* sd, const uint8_t* excluded, int64_t n,
                           int af, double best_std, double lambda, double* partial_score,
                           int64_t* partial_pos, int64_t* partial_first, int64_t* partial_cnt,
                           unsigned int* counter, SelectDev* out, cudaStream_t s) {
  count_launch();
  SelCtx c{mu, nullptr, sd, nullptr, excluded, nullptr, 0, n, 1u << af,
           partial_score, partial_pos, partial_first, partial_cnt, counter, out};
  k_best_candidate<<<reduce_blocks(n), kReduceThreads, 0, s>>>(c, best_std, lambda);
}

void launch_scores(const double* mu, const double* sd, int64_t n, int af, double best_std,
                   double lambda, double* out, cudaStream_t s) {
  count_launch();
  k_scores<<<reduce_blocks(n), kReduceThreads, 0, s>>>(mu, sd, n, af, best_std, lambda, out);
}

}  // namespace gtc
