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
// each valid observation appends ONE row of L (single CTA, bordered Cholesky,
// k_gp_append) and ONE row of V (k_extend<1>): per candidate the new row is
//   v_n = (k(x_n, x*) - sum_{m<n} L_nm v_m) / L_nn
// which is exactly the last step of the reference's forward substitution, and
// the posterior falls out of the same pass:
//   mu = sum_i v_i beta_i  (beta = L^-1 y_standardized),  var = max(s2 - sum_i v_i^2, 0).
// The pass streams V once (HBM-bound GEMV): tile-major V, 16-byte streaming
// loads, 8 rows in flight per thread; its epilogue leaves per-tile partial
// sums of the posterior variance.  The selection (k_select) reduces those
// partials in every block (same fixed order -> same lambda everywhere), then
// EI/PI/LCB + masked argmax in one pass over the candidates.
//
// L is stored packed row-major (row i at i(i+1)/2) so that the whole factor
// of a budget-220 run (194 KB) fits in the shared memory of the single-CTA
// update kernels.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <atomic>
#include <cstdint>
#include <mutex>

#include "gtc_internal.h"

namespace cg = cooperative_groups;

namespace gtc {

static std::atomic<uint64_t> g_launches{0};
uint64_t launches() { return g_launches.load(); }
static inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

__host__ __device__ __forceinline__ int64_t packed(int64_t i) { return i * (i + 1) / 2; }

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

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ long long block_sum_ll(long long v, long long* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum_ll(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  long long t = lane < nw ? red[lane] : 0;
  return warp_sum_ll(t);
}

__device__ __forceinline__ bool visited_bit(const uint32_t* visited, int64_t j) {
  return (__ldg(visited + (j >> 5)) >> (j & 31)) & 1u;
}

// Solves L x = b in place (x in shared memory, length n) with one CTA, using
// the first n rows of the packed lower factor Lp (shared or global memory).
// Forward substitution in the reference's order: every row subtracts its
// terms in ascending column order, then divides by its pivot (as a multiply
// by the pre-computed reciprocal, <= 1 ulp).  This order keeps chosen
// configurations identical to the reference's; a blocked inverse variant
// (explicit diagonal-block inverses + refinement) moved results by ~1e-13
// and flipped near-tied picks, so it is not used.
//
// Row ownership: thread t owns rows t, t+256, t+512, t+768 and keeps their
// running values in registers, so every row is updated by exactly one thread
// and only the 32-step diagonal chain of each block is serial.  Block b's rows
// belong to warp b % 8, which preloads its diagonal block (and pivot
// reciprocals) for its next block while other warps run their chains.
constexpr int kSolveRowsPerThread = kMaxNmax / kCtaThreads;

__device__ __forceinline__ double pick_row(const double (&xo)[kSolveRowsPerThread], int s) {
  double v = xo[0];
#pragma unroll
  for (int q = 1; q < kSolveRowsPerThread; ++q) v = s == q ? xo[q] : v;
  return v;
}

__device__ void cta_forward_solve(const double* Lp, int n, double* x) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = kCtaThreads / 32;
  double xo[kSolveRowsPerThread];
#pragma unroll
  for (int s = 0; s < kSolveRowsPerThread; ++s) {
    const int r = threadIdx.x + s * kCtaThreads;
    xo[s] = r < n ? x[r] : 0.0;
  }
  const int nblk = (n + 31) / 32;
  double lr[32];
  double rinv = 0.0;
  auto load_diag = [&](int blk) {
    const int b0 = blk * 32, r = b0 + lane;
    const bool live = blk < nblk && r < n;
    const double* Lr = Lp + packed(live ? r : 0);
#pragma unroll
    for (int k = 0; k < 32; ++k) lr[k] = (live && k <= lane) ? Lr[b0 + k] : 0.0;
    rinv = live ? __drcp_rn(Lr[r]) : 0.0;
  };
  load_diag(warp);
  for (int blk = 0; blk < nblk; ++blk) {
    const int b0 = blk * 32, b1 = min(b0 + 32, n);
    if (warp == blk % nwarps) {
      const int slot = blk / nwarps;
      double xr = pick_row(xo, slot);
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (b0 + k < b1) {
          if (lane == k) xr = __dmul_rn(xr, rinv);
          const double xi = __shfl_sync(0xffffffffu, xr, k);
          if (lane > k) xr = __dadd_rn(xr, -__dmul_rn(lr[k], xi));
        }
      }
      if (b0 + lane < b1) x[b0 + lane] = xr;
#pragma unroll
      for (int s = 0; s < kSolveRowsPerThread; ++s)
        if (s == slot) xo[s] = xr;
      load_diag(blk + nwarps);  // off the critical path: next owned block
    }
    __syncthreads();  // block b's solution visible
#pragma unroll
    for (int s = 0; s < kSolveRowsPerThread; ++s) {
      const int r = threadIdx.x + s * kCtaThreads;
      if (r >= b1 && r < n) {
        const double* Lr = Lp + packed(r);
        double acc = xo[s];
        for (int i = b0; i < b1; ++i) acc = __dadd_rn(acc, -__dmul_rn(Lr[i], x[i]));
        xo[s] = acc;
      }
    }
  }
  __syncthreads();
}

// Standardisation + beta for the first n observations (gp.hpp:97-103,130).
// Deterministic block-tree sums (fixed order for a given n).
__device__ void cta_stats_beta(const GpDev& g, int n, double* red) {
  __shared__ double s_y0;
  double part = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) part = __dadd_rn(part, g.y[i]);
  const double sum = block_sum(part, red);
  const double mean = n > 0 ? __ddiv_rn(sum, (double)n) : 0.0;
  part = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double dv = __dadd_rn(g.y[i], -mean);
    part = __dadd_rn(part, __dmul_rn(dv, dv));
  }
  const double ss = block_sum(part, red);
  double stdv = 1.0;
  if (n > 1) {
    const double var = __ddiv_rn(ss, (double)n);
    stdv = var > 0.0 ? sqrt(var) : 1.0;
  }
  if (threadIdx.x == 0) {
    s_y0 = g.sc->y0;
    g.sc->y_mean = mean;
    g.sc->y_std = stdv;
    g.sc->n = n;
  }
  __syncthreads();
  const double s_mean = mean, s_std = stdv;
  const double shift = __dadd_rn(s_mean, -s_y0);
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

// Shared-memory layout of the single-CTA GP kernels:
//   xs  work vector (n_max)
//   ys  y copy      (n_max)
//   Ls  packed L rows [0, rows) (staged when they fit, else read from global)
struct CtaSmem {
  double* Ls;
  double* xs;
  double* ys;
  bool staged;
};

__host__ __device__ __forceinline__ int64_t even_up(int64_t v) { return (v + 1) & ~int64_t(1); }
__host__ __device__ __forceinline__ int64_t staged_l_doubles(int rows) { return even_up(packed(rows)); }

__device__ CtaSmem cta_smem_layout(double* base, int n_max, int rows, bool staged) {
  CtaSmem m;
  m.staged = staged;
  m.xs = base;
  m.ys = base + n_max;
  m.Ls = base + even_up(2 * (int64_t)n_max);
  (void)rows;
  return m;
}

__device__ __forceinline__ const double* lp_of(const GpDev& g, const CtaSmem& m) { return m.staged ? m.Ls : g.L; }

// Appends training point `row` (coords already in g.train_x[row]) to the
// factor: l = L^-1 g, pivot = k(0) + noise + jitter - |l|^2 (gp.hpp:105-121).
// Returns false (and records the failure) when the pivot is <= 0.
template <int NU>
__device__ bool cta_border_row(const GpDev& g, KernelParams k, double noise, double jitter, int row,
                               const CtaSmem& m, double* red, unsigned long long* tm = nullptr) {
  const double* xr = g.train_x + (int64_t)row * g.d;
  for (int q = threadIdx.x; q < row; q += blockDim.x)
    m.xs[q] = direct_kernel<NU>(g.train_x + (int64_t)q * g.d, xr, g.d, k.lengthscale, k.s2);
  __syncthreads();
  if (tm && threadIdx.x == 0) tm[2] = gtc_globaltimer();
  cta_forward_solve(lp_of(g, m), row, m.xs);
  if (tm && threadIdx.x == 0) tm[3] = gtc_globaltimer();
  double part = 0.0;
  for (int q = threadIdx.x; q < row; q += blockDim.x) part = __dadd_rn(part, __dmul_rn(m.xs[q], m.xs[q]));
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
  double* Lrow = g.L + packed(row);
  const double lnn = sqrt(x);
  for (int q = threadIdx.x; q < row; q += blockDim.x) {
    Lrow[q] = m.xs[q];
    if (m.staged) m.Ls[packed(row) + q] = m.xs[q];
  }
  if (threadIdx.x == 0) {
    Lrow[row] = lnn;
    if (m.staged) m.Ls[packed(row) + row] = lnn;
  }
  __syncthreads();
  return true;
}

// c[row], e[row] from the new L row (prefix-stable forward substitution).
__device__ void cta_ce_row(const GpDev& g, int row, const CtaSmem& m, double* red) {
  const double* Lrow = lp_of(g, m) + packed(row);
  double pc = 0.0, pe = 0.0;
  for (int q = threadIdx.x; q < row; q += blockDim.x) {
    pc = __dadd_rn(pc, __dmul_rn(Lrow[q], g.c[q]));
    pe = __dadd_rn(pe, __dmul_rn(Lrow[q], g.e[q]));
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

// Rows [0, rows) of the packed factor into shared memory with TMA bulk copies
// (cp.async.bulk global->shared, completion on an mbarrier): the factor is
// evicted from L2 by every V stream, and one SM pulling 194 KB with scalar
// loads is latency-bound; the bulk engine streams it at full rate.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  constexpr uint32_t kChunk = 32768;
  const char* s = reinterpret_cast<const char*>(src);
  for (uint32_t off = 0; off < bytes; off += kChunk) {
    const uint32_t sz = bytes - off < kChunk ? bytes - off : kChunk;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst + off),
                 "l"(s + off), "r"(sz), "r"(bar)
                 : "memory");
  }
}

// Stages L rows [0, l_rows) (size rounded to 16 bytes; the allocation is padded).
__device__ void cta_stage_L(const GpDev& g, int l_rows, const CtaSmem& m) {
  __shared__ __align__(8) uint64_t bar;
  const uint32_t lbytes = static_cast<uint32_t>(staged_l_doubles(l_rows) * 8);
  if (!m.staged || lbytes == 0) {
    __syncthreads();
    return;
  }
  const uint32_t b = smem_u32(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(lbytes) : "memory");
    bulk_g2s(smem_u32(m.Ls), g.L, lbytes, b);
  }
  __syncthreads();  // barrier initialised before anyone waits on it
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(b)
      : "memory");
}

// ------------------------------------------------------------ GP kernels

template <int NU>
__global__ void __launch_bounds__(kCtaThreads)
    k_gp_factor(GpDev g, KernelParams k, double noise, double jitter, int n, int staged) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  const CtaSmem m = cta_smem_layout(smem, g.n_max, n, staged != 0);  // built in place, nothing to stage
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
    if (!cta_border_row<NU>(g, k, noise, jitter, row, m, red)) {
      if (threadIdx.x == 0) g.sc->n = 0;
      return;
    }
  }
  for (int row = 0; row < n; ++row) cta_ce_row(g, row, m, red);
  cta_stats_beta(g, n, red);
}

template <int NU>
__global__ void __launch_bounds__(kCtaThreads)
    k_gp_append(GpDev g, KernelParams k, double noise, SpaceDev sp, int64_t pos,
                const double* x_explicit, double y_new, int n0, uint32_t* visited_mark, int staged) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  __shared__ double xnew[64];
  const CtaSmem m = cta_smem_layout(smem, g.n_max, n0 + 1, staged != 0);
  unsigned long long* tm = g.sc->t;
  if (threadIdx.x == 0) tm[0] = gtc_globaltimer();
  if (visited_mark && threadIdx.x == 0) visited_mark[pos >> 5] |= 1u << (pos & 31);
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
  cta_stage_L(g, n0, m);  // includes __syncthreads
  if (threadIdx.x == 0) {
    tm[1] = gtc_globaltimer();
    double s = 0.0;
    for (int t = 0; t < g.d; ++t) s = __dadd_rn(s, __dmul_rn(xnew[t], xnew[t]));
    g.train_n2[n0] = s;
  }
  const double jitter = g.sc->jitter;
  if (!cta_border_row<NU>(g, k, noise, jitter, n0, m, red, tm)) return;
  if (threadIdx.x == 0) tm[4] = gtc_globaltimer();
  cta_ce_row(g, n0, m, red);
  if (threadIdx.x == 0) tm[5] = gtc_globaltimer();
  cta_stats_beta(g, n0 + 1, red);
  if (threadIdx.x == 0) tm[6] = gtc_globaltimer();
}

__global__ void k_gp_truncate(GpDev g, int n) {
  __shared__ double red[32];
  cta_stats_beta(g, n, red);
}

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
  const uint32_t* visited;  // with part_sum: per-tile variance partials (final pass)
  double* part_sum;
  long long* part_cnt;
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
  double* Ls = sm;              // [R][ld] coefficients of the new rows
  double* bs = sm + R * ld;     // [n0 + r] beta
  double* xn = bs + ld;         // [R][d] new training coords
  double* xn2 = xn + R * a.g.d; // [R] their squared norms
  for (int idx = threadIdx.x; idx < r * (n0 + r); idx += blockDim.x) {
    const int t = idx / (n0 + r), q = idx % (n0 + r);
    Ls[t * ld + q] = q <= n0 + t ? a.g.L[packed(n0 + t) + q] : 0.0;
  }
  if (a.final_pass)
    for (int q = threadIdx.x; q < n0 + r; q += blockDim.x) bs[q] = a.g.beta[q];
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
    const double var0 = fmax(__dadd_rn(a.s2, -q0), 0.0), var1 = fmax(__dadd_rn(a.s2, -q1), 0.0);
    *reinterpret_cast<double2*>(a.mu + j0) = make_double2(b0, b1);
    *reinterpret_cast<double2*>(a.var + j0) = make_double2(var0, var1);
    if (a.part_sum) {
      // this tile's share of the mean posterior variance over the unvisited
      // candidates (strategies.hpp:406-407); plain stores, consumed by the
      // next kernel on the stream (k_select), so no fence is needed
      __shared__ double red[32];
      __shared__ long long redl[32];
      const uint32_t w = j0 < a.sp.n ? __ldg(a.visited + (j0 >> 5)) : 0xffffffffu;
      const bool u0 = j0 < a.sp.n && !((w >> (j0 & 31)) & 1u);
      const bool u1 = j0 + 1 < a.sp.n && !((w >> ((j0 + 1) & 31)) & 1u);
      const double ts = block_sum((u0 ? var0 : 0.0) + (u1 ? var1 : 0.0), red);
      const long long tc = block_sum_ll((long long)u0 + (long long)u1, redl);
      if (threadIdx.x == 0) {
        a.part_sum[blockIdx.x] = ts;
        a.part_cnt[blockIdx.x] = tc;
      }
    }
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

// SM count of the current device (cached per device).
static int sm_count() {
  static std::mutex mu;
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  int& c = cached[dev & 63];
  if (c == 0) {
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    if (c <= 0) c = 148;
  }
  return c;
}

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

// Per-block partial of the variance sum over unvisited candidates (strided,
// fixed order), returned by every thread.
__device__ void var_partial(const double* __restrict__ var, const uint32_t* __restrict__ visited,
                            int64_t n, double* red, long long* redl, double* out_sum, long long* out_cnt) {
  double s = 0.0;
  long long c = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (!visited_bit(visited, j)) {
      s += var[j];
      ++c;
    }
  }
  *out_sum = block_sum(s, red);
  *out_cnt = block_sum_ll(c, redl);
}

// Deterministic fixed-order sum of `count` block partials, in every block.
__device__ void reduce_partials(const double* ps, const long long* pc, int count, double* red,
                                long long* redl, double* sum, long long* cnt) {
  // four independent accumulators keep four loads in flight per thread
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  long long c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  const int bd = blockDim.x;
  int b = threadIdx.x;
  for (; b + 3 * bd < count; b += 4 * bd) {
    const double p0 = __ldcg(ps + b), p1 = __ldcg(ps + b + bd), p2 = __ldcg(ps + b + 2 * bd), p3 = __ldcg(ps + b + 3 * bd);
    const long long q0 = __ldcg(pc + b), q1 = __ldcg(pc + b + bd), q2 = __ldcg(pc + b + 2 * bd), q3 = __ldcg(pc + b + 3 * bd);
    s0 += p0; s1 += p1; s2 += p2; s3 += p3;
    c0 += q0; c1 += q1; c2 += q2; c3 += q3;
  }
  for (; b < count; b += bd) {
    s0 += __ldcg(ps + b);
    c0 += __ldcg(pc + b);
  }
  *sum = block_sum((s0 + s1) + (s2 + s3), red);
  *cnt = block_sum_ll((c0 + c1) + (c2 + c3), redl);
}

__global__ void __launch_bounds__(kReduceThreads)
    k_varsum(const double* __restrict__ var, const uint32_t* __restrict__ visited, int64_t n,
             double* partial_sum, int64_t* partial_cnt, unsigned int* counter, VarTotals* totals) {
  __shared__ double red[32];
  __shared__ long long redl[32];
  double s;
  long long c;
  var_partial(var, visited, n, red, redl, &s, &c);
  if (threadIdx.x == 0) {
    partial_sum[blockIdx.x] = s;
    partial_cnt[blockIdx.x] = c;
  }
  if (!last_block(counter)) return;
  reduce_partials(partial_sum, reinterpret_cast<const long long*>(partial_cnt), gridDim.x, red, redl, &s, &c);
  if (threadIdx.x == 0) {
    totals->sum = s;
    totals->count = c;
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
  ReduceBufs b;
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

template <uint32_t MASK>
__device__ __forceinline__ void score_into(Best* b, double m, double sd, double best, double lambda, int64_t j) {
#pragma unroll
  for (int af = 0; af < 3; ++af) {
    if (!(MASK & (1u << af))) continue;
    const double s = score_of(af, m, sd, best, lambda);
    if (s == s) b[af] = better(b[af], Best{s, j});
  }
}

// Block reduction of the per-thread (best per AF, first eligible, count)
// followed by the last-block merge into the result record.
template <uint32_t MASK>
__device__ void select_finish(const SelCtx& c, Best* b, int64_t first, long long cnt, double best,
                              double lambda, double mean_var, int cv_fallback, int gp_status) {
  __shared__ Best redb[32];
  __shared__ int64_t redi[32];
  __shared__ long long redl[32];
  cnt = block_sum_ll(cnt, redl);
#pragma unroll
  for (int af = 0; af < 3; ++af)
    if (MASK & (1u << af)) b[af] = block_best(b[af], redb);
  first = block_min(first, redi);
  if (threadIdx.x == 0) {
    for (int af = 0; af < 3; ++af) {
      c.b.pscore[blockIdx.x * 3 + af] = b[af].s;
      c.b.ppos[blockIdx.x * 3 + af] = b[af].p;
    }
    c.b.pfirst[blockIdx.x] = first;
    c.b.pcnt[blockIdx.x] = cnt;
  }
  if (!last_block(c.b.counter)) return;
  Best f[3] = {{0.0, INT64_MAX}, {0.0, INT64_MAX}, {0.0, INT64_MAX}};
  int64_t ff = INT64_MAX;
  long long fc = 0;
  for (int blk = threadIdx.x; blk < gridDim.x; blk += blockDim.x) {
    for (int af = 0; af < 3; ++af)
      f[af] = better(f[af], Best{__ldcg(c.b.pscore + blk * 3 + af),
                                 (int64_t)__ldcg(reinterpret_cast<const long long*>(c.b.ppos) + blk * 3 + af)});
    ff = min(ff, (int64_t)__ldcg(reinterpret_cast<const long long*>(c.b.pfirst) + blk));
    fc += __ldcg(c.b.pcnt + blk);
  }
  for (int af = 0; af < 3; ++af) f[af] = block_best(f[af], redb);
  ff = block_min(ff, redi);
  fc = block_sum_ll(fc, redl);
  if (threadIdx.x == 0) {
    c.out->first_nan_mask = 0;
    for (int af = 0; af < 3; ++af) {
      c.out->best_nonnan_pos[af] = -1;
      c.out->best_nonnan_score[af] = 0.0;
    }
    for (int af = 0; af < 3; ++af) {
      int64_t pos = -1;
      double sc = 0.0;
      if ((c.af_mask & (1u << af)) && fc > 0) {
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
        // the pieces a cross-shard merge needs to apply the same rule
        c.out->best_nonnan_pos[af] = f[af].p == INT64_MAX ? -1 : f[af].p;
        c.out->best_nonnan_score[af] = f[af].s;
        if (s_first != s_first) c.out->first_nan_mask |= 1u << af;
      }
      c.out->position[af] = pos;
      c.out->score[af] = sc;
    }
    c.out->first_eligible = fc > 0 ? ff : -1;
    c.out->lambda = lambda;
    c.out->mean_variance = mean_var;
    c.out->best_std = best;
    c.out->n_candidates = (int64_t)fc;
    c.out->cv_fallback = cv_fallback;
    c.out->gp_status = gp_status;
    *c.b.counter = 0;
  }
}

// Scan of a strided slice: software-pipelined (the next candidate's visited
// word, mean and variance/std are in flight while the current one is scored;
// one copy of the erfc/exp code keeps the loop in the instruction cache).
// Shared by the run selection and the span-based best_candidate path.
template <uint32_t MASK>
__device__ void select_body(const SelCtx& c, double best, double lambda, double mean_var,
                            int cv_fallback, int gp_status) {
  Best b[3] = {{0.0, INT64_MAX}, {0.0, INT64_MAX}, {0.0, INT64_MAX}};
  int64_t first = INT64_MAX;
  long long cnt = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double* spread = c.sdv ? c.sdv : c.var;
  bool e_cur = false;
  double m_cur = 0.0, v_cur = 0.0;
  if (j < c.n) {
    e_cur = eligible(c, j);
    m_cur = c.mu[j];
    v_cur = spread[j];
  }
#pragma unroll 1
  for (; j < c.n; j += stride) {
    const int64_t jn = j + stride;
    bool e_nxt = false;
    double m_nxt = 0.0, v_nxt = 0.0;
    if (jn < c.n) {
      e_nxt = eligible(c, jn);
      m_nxt = c.mu[jn];
      v_nxt = spread[jn];
    }
    if (e_cur) {
      ++cnt;
      first = min(first, j);
      // cand_stds = sqrt(cand_vars), strategies.hpp:385
      score_into<MASK>(b, m_cur, c.sdv ? v_cur : sqrt(v_cur), best, lambda, j);
    }
    e_cur = e_nxt;
    m_cur = m_nxt;
    v_cur = v_nxt;
  }
  select_finish<MASK>(c, b, first, cnt, best, lambda, mean_var, cv_fallback, gp_status);
}

// Selection for a resident run.  The mean posterior variance over the
// unvisited candidates comes from the per-tile partials the predictive pass
// (or k_var_partials) left behind: every block reduces the same `n_partials`
// values in the same fixed order, so all blocks agree on lambda
// (strategies.hpp:404-418, acquisition.hpp:73-83) and best_std (gp.hpp:145)
// without a grid barrier; then the masked argmax as in select_body.
template <uint32_t MASK>
__global__ void __launch_bounds__(kSelectThreads, 1)
    k_select(SelCtx c, const GpScalars* sc, SelectParams p, const double* part_sum,
             const long long* part_cnt, int n_partials) {
  __shared__ double red[32];
  __shared__ long long redl[32];
  double s;
  long long cnt;
  reduce_partials(part_sum, part_cnt, n_partials, red, redl, &s, &cnt);
  const double mean_var = cnt > 0 ? __ddiv_rn(s, (double)cnt) : 0.0;
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
  select_body<MASK>(c, best, lambda, mean_var, fallback, sc->status);
}

// Total of a partials array (one block, fixed order): a shard's local
// contribution to the global mean variance.
__global__ void __launch_bounds__(kReduceThreads)
    k_reduce_partials(const double* part_sum, const long long* part_cnt, int n_partials, VarTotals* out) {
  __shared__ double red[32];
  __shared__ long long redl[32];
  double s;
  long long c;
  reduce_partials(part_sum, part_cnt, n_partials, red, redl, &s, &c);
  if (threadIdx.x == 0) {
    out->sum = s;
    out->count = c;
  }
}

// Variance partials over the unvisited candidates when the pass did not
// produce them for the current visited set (invalid observation, unmark).
__global__ void __launch_bounds__(kReduceThreads)
    k_var_partials(const double* __restrict__ var, const uint32_t* __restrict__ visited, int64_t n,
                   double* part_sum, long long* part_cnt) {
  __shared__ double red[32];
  __shared__ long long redl[32];
  double s;
  long long c;
  var_partial(var, visited, n, red, redl, &s, &c);
  if (threadIdx.x == 0) {
    part_sum[blockIdx.x] = s;
    part_cnt[blockIdx.x] = c;
  }
}

template <uint32_t MASK>
__global__ void __launch_bounds__(kReduceThreads) k_best_candidate(SelCtx c, double best, double lambda) {
  select_body<MASK>(c, best, lambda, 0.0, 0, 0);
}

__global__ void k_scores(const double* __restrict__ mu, const double* __restrict__ sd, int64_t n,
                         int af, double best, double lambda, double* out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = score_of(af, mu[j], sd[j], best, lambda);
}

// ------------------------------------------------------------ launchers

// Shared memory of the single-CTA GP kernels: xs + ys (+ packed L rows and
// diagonal-block inverses when they fit under the opt-in limit).
static size_t cta_smem_bytes(int n_max, int rows, bool* staged) {
  const size_t base = sizeof(double) * (size_t)even_up(2 * (int64_t)n_max);
  const size_t with_l = base + sizeof(double) * (size_t)staged_l_doubles(rows);
  *staged = with_l <= kCtaSmemLimit;
  return *staged ? with_l : base;
}

template <class K>
static void opt_in_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

void launch_gp_factor(const GpDev& g, KernelParams k, double noise, double jitter, int n,
                      cudaStream_t s) {
  count_launch();
  bool staged;
  const size_t sm = cta_smem_bytes(g.n_max, n, &staged);
  const int st = staged ? 1 : 0;
  switch (k.nu) {
    case 0: opt_in_smem(k_gp_factor<0>, sm); k_gp_factor<0><<<1, kCtaThreads, sm, s>>>(g, k, noise, jitter, n, st); break;
    case 1: opt_in_smem(k_gp_factor<1>, sm); k_gp_factor<1><<<1, kCtaThreads, sm, s>>>(g, k, noise, jitter, n, st); break;
    default: opt_in_smem(k_gp_factor<2>, sm); k_gp_factor<2><<<1, kCtaThreads, sm, s>>>(g, k, noise, jitter, n, st); break;
  }
}

void launch_gp_append(const GpDev& g, KernelParams k, double noise, const SpaceDev& sp,
                      int64_t pos, const double* x_explicit, double y_new, int n0,
                      uint32_t* visited_mark, cudaStream_t s) {
  count_launch();
  bool staged;
  const size_t sm = cta_smem_bytes(g.n_max, n0 + 1, &staged);
  const int st = staged ? 1 : 0;
  switch (k.nu) {
    case 0: opt_in_smem(k_gp_append<0>, sm); k_gp_append<0><<<1, kCtaThreads, sm, s>>>(g, k, noise, sp, pos, x_explicit, y_new, n0, visited_mark, st); break;
    case 1: opt_in_smem(k_gp_append<1>, sm); k_gp_append<1><<<1, kCtaThreads, sm, s>>>(g, k, noise, sp, pos, x_explicit, y_new, n0, visited_mark, st); break;
    default: opt_in_smem(k_gp_append<2>, sm); k_gp_append<2><<<1, kCtaThreads, sm, s>>>(g, k, noise, sp, pos, x_explicit, y_new, n0, visited_mark, st); break;
  }
}

void launch_gp_truncate(const GpDev& g, int n, cudaStream_t s) {
  count_launch();
  k_gp_truncate<<<1, kCtaThreads, 0, s>>>(g, n);
}

template <int R, int NU>
static void extend_impl(const ExtendArgs& a, int64_t tiles, cudaStream_t s) {
  const size_t sm = sizeof(double) * ((size_t)(R + 1) * (a.n0 + R) + (size_t)R * a.g.d + R + 8);
  opt_in_smem(k_extend<R, NU>, sm);
  k_extend<R, NU><<<(unsigned)tiles, kExtendThreads, sm, s>>>(a);
}

void launch_extend(const SpaceDev& sp, const GpDev& g, KernelParams k, double* V,
                   int64_t tile_stride, int n0, int r, bool final, double* mu, double* var,
                   bool check_status, const VarPartials* vp, cudaStream_t s) {
  count_launch();
  ExtendArgs a{sp, g, V, tile_stride, n0, r, final ? 1 : 0, check_status ? 1 : 0,
               k.lengthscale, k.s2, mu, var, vp ? vp->visited : nullptr,
               (vp && final) ? vp->part_sum : nullptr, vp ? vp->part_cnt : nullptr};
  const int64_t tiles = sp.n_pad / kTile;
  if (r <= 1) {
    switch (k.nu) {
      case 0: extend_impl<1, 0>(a, tiles, s); break;
      case 1: extend_impl<1, 1>(a, tiles, s); break;
      default: extend_impl<1, 2>(a, tiles, s); break;
    }
  } else {
    switch (k.nu) {
      case 0: extend_impl<kMaxRows, 0>(a, tiles, s); break;
      case 1: extend_impl<kMaxRows, 1>(a, tiles, s); break;
      default: extend_impl<kMaxRows, 2>(a, tiles, s); break;
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

void launch_reduce_partials(const double* part_sum, const long long* part_cnt, int n_partials, VarTotals* out,
                            cudaStream_t s) {
  count_launch();
  k_reduce_partials<<<1, kReduceThreads, 0, s>>>(part_sum, part_cnt, n_partials, out);
}

void launch_var_partials(const double* var, const uint32_t* visited, int64_t n, double* part_sum,
                         long long* part_cnt, cudaStream_t s) {
  count_launch();
  k_var_partials<<<reduce_blocks(n), kReduceThreads, 0, s>>>(var, visited, n, part_sum, part_cnt);
}

void launch_select(const double* mu, const double* var, const uint32_t* visited, int64_t n,
                   const GpScalars* sc, SelectParams p, const double* part_sum, const long long* part_cnt,
                   int n_partials, const ReduceBufs& b, SelectDev* out, cudaStream_t s) {
  count_launch();
  SelCtx c{mu, var, nullptr, visited, nullptr, p.excluded, p.n_excluded, n, p.af_mask, b, out};
  // exactly one wave of resident blocks (grid-stride inside): a partial
  // second wave would double the kernel's time
  const int per_block = kSelectThreads * 2;
  int grid = (int)std::min<int64_t>((n + per_block - 1) / per_block, (int64_t)sm_count());
  grid = std::max(std::min(grid, kMaxReduceGrid), 1);
#define GTC_SELECT_CASE(M) \
  case M: k_select<M><<<grid, kSelectThreads, 0, s>>>(c, sc, p, part_sum, part_cnt, n_partials); break;
  switch (p.af_mask & 7u) {  // launch errors surface through the caller's cudaGetLastError()
    GTC_SELECT_CASE(1)
    GTC_SELECT_CASE(2)
    GTC_SELECT_CASE(3)
    GTC_SELECT_CASE(4)
    GTC_SELECT_CASE(5)
    GTC_SELECT_CASE(6)
    default: k_select<7><<<grid, kSelectThreads, 0, s>>>(c, sc, p, part_sum, part_cnt, n_partials); break;
  }
#undef GTC_SELECT_CASE
}

void launch_best_candidate(const double* mu, const double* sd, const uint8_t* excluded, int64_t n,
                           int af, double best_std, double lambda, const ReduceBufs& b, SelectDev* out,
                           cudaStream_t s) {
  count_launch();
  SelCtx c{mu, nullptr, sd, nullptr, excluded, nullptr, 0, n, 1u << af, b, out};
  const int grid = reduce_blocks(n);
  if (af == 0) k_best_candidate<1><<<grid, kReduceThreads, 0, s>>>(c, best_std, lambda);
  else if (af == 1) k_best_candidate<2><<<grid, kReduceThreads, 0, s>>>(c, best_std, lambda);
  else k_best_candidate<4><<<grid, kReduceThreads, 0, s>>>(c, best_std, lambda);
}

void launch_scores(const double* mu, const double* sd, int64_t n, int af, double best_std,
                   double lambda, double* out, cudaStream_t s) {
  count_launch();
  k_scores<<<reduce_blocks(n), kReduceThreads, 0, s>>>(mu, sd, n, af, best_std, lambda, out);
}

}  // namespace gtc
