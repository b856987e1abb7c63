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
// loads, 6 rows in flight per thread, 1-byte coordinate indices; its epilogue
// adds the tile's variance sum to a fixed-point total (VarAccum) and records
// a per-tile posterior summary (TileStats).  The selection (k_select) reads
// the total (same lambda in every block), bounds tiles and candidates with
// rigorous FP32 Mills-ratio keys and scores exactly in FP64 only what can
// reach a threshold (see the "pruned selection" section).
//
// L is stored packed row-major (row i at i(i+1)/2) so that the whole factor
// of a budget-220 run (194 KB) fits in the shared memory of the single-CTA
// update kernels.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "gtc_internal.h"

namespace cg = cooperative_groups;

namespace gtc {

#ifdef GTC_SEL_TRACE  // diagnostic per-block %globaltimer marks (tools/sel_bench.cu)
__device__ unsigned long long g_sel_trace[2048][8];
#define SEL_MARK(k) \
  do { if (threadIdx.x == 0) g_sel_trace[blockIdx.x][k] = gtc_globaltimer(); } while (0)
#define TRACE_AT(row, k) \
  do { if (threadIdx.x == 0) g_sel_trace[row][k] = gtc_globaltimer(); } while (0)
#else
#define SEL_MARK(k) do {} while (0)
#define TRACE_AT(row, k) do {} while (0)
#endif

// Diagnostics (GTC_SEL_TRACE builds only): the %globaltimer marks of the
// last selection (rows = blocks; marks 0-3, 5 per block, 6 in the last
// block), the loop-mode append (row 2040) and the pass (row 2041, block 0).
int read_sel_trace(unsigned long long* out, int rows) {
#ifdef GTC_SEL_TRACE
  return cudaMemcpyFromSymbol(out, g_sel_trace, sizeof(unsigned long long) * 8 * (size_t)rows) == cudaSuccess ? 0 : -4;
#else
  (void)out;
  (void)rows;
  return -1;
#endif
}

static std::atomic<uint64_t> g_launches{0};
uint64_t launches() { return g_launches.load(); }
static inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Programmatic dependent launch (resident loop): let the next kernel of the
// stream be scheduled now, then wait until every preceding kernel has
// completed and its writes are visible.  Both are no-ops for a kernel
// launched without the PDL attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_begin() {
  pdl_trigger();
  pdl_wait();
}

// Per host thread: whether launch_pdl sets the PDL attribute (gtc_run_set_pdl;
// off for runs that share the device with many concurrent streams, where
// early-launched waiting CTAs would take SM slots from the other streams).
static thread_local bool t_pdl = true;
void set_thread_pdl(bool on) { t_pdl = on; }

// cudaLaunchKernelEx with programmatic stream serialisation.
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  if (!t_pdl) {
    kernel<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

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

// a / b correctly rounded (== __ddiv_rn) from the correctly rounded
// reciprocal y = 1/b: one Markstein correction step (r = a - q0 b is exact by
// FMA).  Outside the safe exponent range (and for a == 0, keeping the sign
// of zero) it defers to __ddiv_rn.  Checked bit for bit against __ddiv_rn
// on 1.7e10 operand pairs of the rebuild's ranges (tools/div_check.cu).
__device__ __noinline__ double ddiv_slow(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ double quot_rn(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double aq = fabs(q0), aa = fabs(a);
  if (!(aq < 0x1p+960 && aq > 0x1p-960 && aa > 0x1p-960 && aa < 0x1p+960)) return __ddiv_rn(a, b);
  const double r = fma(-q0, b, a);
  return fma(r, y, q0);
}

// quot_rn with the out-of-range case out of line (compact code for the
// heavily unrolled tensor-core passes: their instruction-cache misses were
// the top stall)
__device__ __forceinline__ double quot_rn_c(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double aq = fabs(q0), aa = fabs(a);
  if (!(aq < 0x1p+960 && aq > 0x1p-960 && aa > 0x1p-960 && aa < 0x1p+960)) return ddiv_slow(a, b);
  const double r = fma(-q0, b, a);
  return fma(r, y, q0);
}

// matern<NU> with the distance scaled by quot_rn (the same bits as its
// __ddiv_rn(r, lengthscale)); linv = __drcp_rn(lengthscale).
template <int NU>
__device__ __forceinline__ double matern_q(double r, double lengthscale, double linv, double s2) {
  const double s = quot_rn(r, lengthscale, linv);
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

// Deterministic sums of the O(n) GP vectors that do not depend on the block
// size: element q belongs to virtual lane q % 256 (ascending q within a
// lane), and the 256 lane partials are combined with exactly the tree of
// block_sum in a 256-thread block.  The bordered append runs in 256-thread
// GP kernels and in the selection's last block (128 or 512 threads); with
// these sums both give bit-identical factors.  `lanes[k][256]` hold the lane
// partials (written by the caller before the call); every thread gets out[k].
template <int K>
__device__ void vsum256(double (*lanes)[256], double* out, double* red /* >= 8 K */) {
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int vw = w; vw < 8; vw += nw) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double v = warp_sum(lanes[k][vw * 32 + lane]);
      if (lane == 0) red[k * 8 + vw] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = warp_sum(lane < 8 ? red[k * 8 + lane] : 0.0);
  __syncthreads();  // lanes / red reusable
}

__device__ __forceinline__ bool visited_bit(const uint32_t* visited, int64_t j) {
  return (__ldg(visited + (j >> 5)) >> (j & 31)) & 1u;
}

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// ---- deterministic variance totals (VarAccum, gtc_internal.h) ----
__device__ __forceinline__ int var_scale_exp(double s2) {
  const int e = ilogb(s2);
  return (s2 > 0.0 && e > -900 && e < 900) ? e : 0;
}

// Adds one block's variance sum `ts` (of `tc` candidates, each in [0, s2]).
__device__ void accum_add(VarAccum* a, double ts, long long tc, double s2) {
  double w = ldexp(ts, 120 - var_scale_exp(s2));  // < 2^(121 + log2 tc): fits 4 x 42 bits
#pragma unroll
  for (int k = 3; k >= 0; --k) {
    const double p = floor(ldexp(w, -42 * k));
    w = __dadd_rn(w, -ldexp(p, 42 * k));  // exact: both are multiples of ulp(w)
    if (p != 0.0) atomicAdd(&a->limb[k], (unsigned long long)p);
  }
  if (tc) atomicAdd(&a->count, (unsigned long long)tc);
}

// One candidate's variance in (sign = +1) or out (sign = -1) of a total: the
// visited set changed by one mark, so the total is updated in O(1) instead of
// re-reduced over N.  Limbs are read as signed (two's complement), so a
// subtraction that borrows within a limb is exact.
__device__ void accum_add_one(VarAccum* a, double v, int sign, double s2) {
  double w = ldexp(v, 120 - var_scale_exp(s2));
#pragma unroll
  for (int k = 3; k >= 0; --k) {
    const double p = floor(ldexp(w, -42 * k));
    w = __dadd_rn(w, -ldexp(p, 42 * k));
    const unsigned long long l = (unsigned long long)p;
    if (l) atomicAdd(&a->limb[k], sign > 0 ? l : (unsigned long long)(-(long long)l));
  }
  atomicAdd(&a->count, sign > 0 ? 1ull : (unsigned long long)(-1ll));
}

__device__ __forceinline__ double limbs_value(const unsigned long long* limb, double s2) {
  double t = 0.0;
#pragma unroll
  for (int k = 3; k >= 0; --k) t = __dadd_rn(ldexp(t, 42), (double)(long long)limb[k]);
  return ldexp(t, var_scale_exp(s2) - 120);
}

__device__ __forceinline__ void accum_read(const VarAccum* a, double s2, double* sum, long long* cnt) {
  unsigned long long l[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) l[k] = __ldcg(&a->limb[k]);
  *sum = limbs_value(l, s2);
  *cnt = (long long)__ldcg(&a->count);
}

// Total of the all-gathered shard accumulators (generation `gen` of each):
// integer limb sums (wrapping, two's complement), so the result equals the
// total one device would have accumulated over the union of the tiles.
__device__ __forceinline__ void accum_read_gathered(const VarAccum* g, int n, int gen, double s2, double* sum,
                                                    long long* cnt) {
  unsigned long long l[4] = {0ull, 0ull, 0ull, 0ull}, c = 0ull;
  for (int i = 0; i < n; ++i) {
    const VarAccum* a = g + 2 * i + gen;
#pragma unroll
    for (int k = 0; k < 4; ++k) l[k] += __ldcg(&a->limb[k]);
    c += __ldcg(&a->count);
  }
  *sum = limbs_value(l, s2);
  *cnt = (long long)c;
}

__device__ __forceinline__ void accum_clear(VarAccum* a) {
  if (a && blockIdx.x == 0 && threadIdx.x < 5) reinterpret_cast<unsigned long long*>(a)[threadIdx.x] = 0ull;
}

__device__ __forceinline__ void var_source_read(const VarSource& v, double* sum, long long* cnt) {
  if (v.direct) {
    *sum = v.sum;
    *cnt = v.count;
  } else if (v.gathered) {
    accum_read_gathered(v.gathered, v.n_gathered, v.gen, v.s2, sum, cnt);
  } else {
    accum_read(v.acc, v.s2, sum, cnt);
  }
}

// Solves L x = b in place (x in shared memory, length n) for the first n
// rows of the packed lower factor Lp (shared or global memory), given the
// pivot reciprocals rinv[i] = 1/L_ii (shared).  Forward substitution in the
// reference's order: every row subtracts its terms in ascending column order,
// then multiplies by the pivot reciprocal (<= 1 ulp from the division).  This
// order keeps chosen configurations identical to the reference's; a blocked
// inverse variant (explicit diagonal-block inverses + refinement) moved
// results by ~1e-13 and flipped near-tied picks, so it is not used.
//
// Block-pipelined over 32-row blocks: warp s % 8 runs block s's 32-step
// diagonal chain in registers (shuffle per step, no barrier).  The warp that
// owns block s+1 loads its coefficients (block s+1's diagonal block and block
// s's columns of its rows) while that chain runs, and after one barrier folds
// block s's solution into its rows (one row per lane, the subtractions in
// ascending column order) and goes straight on to the next chain; the other
// warps fold block s into the rows beyond, off the critical path.
constexpr int kSolveWarps = kCtaThreads / 32;

__device__ __forceinline__ void fold_block(const double* Lp, double* x, int r, int b0, int kmax) {
  const double* Lr = Lp + packed(r) + b0;
  double acc = x[r];
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (k < kmax) acc = __dadd_rn(acc, -__dmul_rn(Lr[k], x[b0 + k]));
  x[r] = acc;
}

__device__ void cta_forward_solve(const double* Lp, int n, double* x, const double* rinv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblk = (n + 31) / 32;
  double lrd[32];  // diagonal-block coefficients of the block this warp will chain next
  double lf[32];   // block s's columns of this warp's next rows (fold)
  double xr = 0.0, ri = 0.0;
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
    if (warp == wn && s + 1 < nblk) {  // prefetch while block s's chain runs
      const int r = b0 + 32 + lane;
      const bool live = r < n;
      const double* Lr = Lp + packed(live ? r : b0) + b0;
#pragma unroll
      for (int k = 0; k < 32; ++k) lf[k] = (live && k < kmax) ? Lr[k] : 0.0;
      load_diag(s + 1);
    }
    if (warp == s % kSolveWarps) {  // xr: this warp's rows, complete w.r.t. columns < b0
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
    __syncthreads();  // block s solved; every fold of block s-1 done
    if (s + 1 < nblk) {
      if (warp == wn) {
        const int r = b0 + 32 + lane;
        xr = r < n ? x[r] : 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (k < kmax) xr = __dadd_rn(xr, -__dmul_rn(lf[k], x[b0 + k]));
      } else {
        // far rows on the warps that do not share a scheduler with the next
        // chain (warps wn and wn + 4 share one of the 4 SM sub-partitions)
        const int wo = (wn + kSolveWarps / 2) % kSolveWarps;
        if (warp != wo) {
          const int t = threadIdx.x - 32 * ((warp > wn) + (warp > wo));
          for (int r = b0 + 64 + t; r < n; r += kCtaThreads - 64) fold_block(Lp, x, r, b0, kmax);
        }
      }
    }
  }
  __syncthreads();
}

// Standardisation + beta for the first n observations (gp.hpp:97-103,130).
// Deterministic virtual-lane sums (fixed order for a given n, any block size).
// `ysum`: the sum of y[0, n) when the caller already reduced it (have_ysum).
__device__ void cta_stats_beta(const GpDev& g, int n, bool have_ysum = false, double ysum = 0.0) {
  __shared__ double lanes[1][256];
  __shared__ double red[8];
  __shared__ double s_y0;
  double out[1];
  if (!have_ysum) {
    for (int v = threadIdx.x; v < 256; v += blockDim.x) {
      double part = 0.0;
      for (int i = v; i < n; i += 256) part = __dadd_rn(part, g.y[i]);
      lanes[0][v] = part;
    }
    vsum256<1>(lanes, out, red);
    ysum = out[0];
  }
  const double mean = n > 0 ? __ddiv_rn(ysum, (double)n) : 0.0;
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    double part = 0.0;
    for (int i = v; i < n; i += 256) {
      const double dv = __dadd_rn(g.y[i], -mean);
      part = __dadd_rn(part, __dmul_rn(dv, dv));
    }
    lanes[0][v] = part;
  }
  vsum256<1>(lanes, out, red);
  const double ss = out[0];
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
  const double shift = __dadd_rn(mean, -s_y0);
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    g.beta[i] = __ddiv_rn(__dadd_rn(g.c[i], -__dmul_rn(shift, g.e[i])), stdv);
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
//   xs    work vector (n_max)
//   rinv  pivot reciprocals 1/L_ii of the factor's rows (n_max)
//   Ls  packed L rows [0, rows) (staged when they fit, else read from global)
struct CtaSmem {
  double* Ls;
  double* xs;
  double* rinv;
  bool staged;
};

__host__ __device__ __forceinline__ int64_t even_up(int64_t v) { return (v + 1) & ~int64_t(1); }
__host__ __device__ __forceinline__ int64_t staged_l_doubles(int rows) { return even_up(packed(rows)); }

__device__ CtaSmem cta_smem_layout(double* base, int n_max, int rows, bool staged) {
  CtaSmem m;
  m.staged = staged;
  m.xs = base;
  m.rinv = base + n_max;
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
  cta_forward_solve(lp_of(g, m), row, m.xs, m.rinv);
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
    m.rinv[row] = __drcp_rn(lnn);
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

// Observation n0's training row (coordinates of candidate `pos`, or the
// explicit point when pos < 0), raw value and squared norm; clears the
// factorisation status.  Block-wide; ends with a barrier.
__device__ void append_prologue(const GpDev& g, const SpaceDev& sp, int64_t pos, const double* x_explicit,
                                double y_new, int n0) {
  for (int t = threadIdx.x; t < g.d; t += blockDim.x)
    g.train_x[(int64_t)n0 * g.d + t] = pos >= 0 ? sp.coords[(int64_t)t * sp.n_pad + pos] : x_explicit[t];
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int t = 0; t < g.d; ++t) {
      const double v = g.train_x[(int64_t)n0 * g.d + t];
      s = __dadd_rn(s, __dmul_rn(v, v));
    }
    g.train_n2[n0] = s;
    g.y[n0] = y_new;
    g.sc->status = 0;
    g.sc->fail_row = -1;
    if (n0 == 0) g.sc->y0 = y_new;
  }
  __syncthreads();
}

// Bordered row n0 from the resident V column of the observed candidate.
// The predictive pass already holds, for every candidate x, the forward
// substitution V(:, x) = L^-1 k(X, x) (gp.hpp:163-164) -- which is exactly the
// new row l = L^-1 k(X, x*) of the bordered factor (gp.hpp:105-121 restricted
// to the last row).  The two differ only in how k is rounded: the reference's
// Gram matrix uses direct differences (gp.hpp:110), the cross covariance the
// expansion form (gp.hpp:176-179), both within a few ulp of the exact kernel.
// So the row costs n0 strided loads and three block sums instead of an
// n0-step dependent substitution chain.  The pivot x = k(0) + noise + jitter
// - |l|^2 is a cancellation: when it is below 2^-8 of the diagonal (the
// candidate is close to observed points, where the rounding of l matters
// relative to x, and where the reference's own LLT test x <= 0 may flip) the
// row is left to the exact substitution (returns false, nothing written).
// `col` = V(0, x*), consecutive rows `col_stride` apart.  Block-wide.
// (k(0) = s2 for every nu: the Matern polynomial is 1 and exp(0) = 1 exactly.)
// One fused reduction gives |l|^2, l.c, l.e and the sum of y[0, n0] (the
// standardisation's mean), then cta_stats_beta finishes; all sums are
// virtual-lane sums, so the result does not depend on the block size.
__device__ bool column_border_row(const GpDev& g, KernelParams k, double noise, const double* col,
                                  int64_t col_stride, int n0, double* xs) {
  __shared__ double lanes[4][256];
  __shared__ double red[32];
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    double sq = 0.0, pc = 0.0, pe = 0.0, py = 0.0;
    for (int q = v; q < n0; q += 256) {
      const double l = __ldcg(col + (int64_t)q * col_stride);
      xs[q] = l;
      sq = __dadd_rn(sq, __dmul_rn(l, l));
      pc = __dadd_rn(pc, __dmul_rn(l, g.c[q]));
      pe = __dadd_rn(pe, __dmul_rn(l, g.e[q]));
      py = __dadd_rn(py, g.y[q]);
    }
    if (v == n0 % 256) py = __dadd_rn(py, g.y[n0]);  // the new observation, last in its lane
    lanes[0][v] = sq;
    lanes[1][v] = pc;
    lanes[2][v] = pe;
    lanes[3][v] = py;
  }
  double r[4];
  vsum256<4>(lanes, r, red);
  const double diag = __dadd_rn(k.s2, __dadd_rn(noise, g.sc->jitter));
  const double x = __dadd_rn(diag, -r[0]);
  if (!(x > 0x1p-8 * diag)) return false;
  const double lnn = sqrt(x);
  double* Lrow = g.L + packed(n0);
  for (int q = threadIdx.x; q < n0; q += blockDim.x) Lrow[q] = xs[q];
  if (threadIdx.x == 0) {
    Lrow[n0] = lnn;
    const double yr = __dadd_rn(g.y[n0], -g.sc->y0);
    g.c[n0] = __ddiv_rn(__dadd_rn(yr, -r[1]), lnn);
    g.e[n0] = __ddiv_rn(__dadd_rn(1.0, -r[2]), lnn);
  }
  __syncthreads();
  cta_stats_beta(g, n0 + 1, true, r[3]);
  return true;
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
  cta_stats_beta(g, n);
}

// The same factorisation, right-looking, with the whole packed factor in
// shared memory (n <= ~230): step j takes row j's pivot (|L_j,<j|^2 as the
// 256-lane tree sum of cta_border_row's block_sum), scales column j below
// the diagonal by 1/L_jj and folds column j into the trailing rows.  Every
// entry receives exactly the left-looking operations in the same order --
// acc - L_rk * x_k for ascending k, then times 1/L_rr -- so the factor is
// bit-identical to k_gp_factor's, in n barrier-separated steps instead of
// n dependent substitution chains (O(n^2) latency).  The first failing
// pivot (x <= 0) is the same row.
constexpr int kFactorThreads = 1024;  // the trailing updates are latency-bound: all the warps one CTA can hold

template <int NU>
__global__ void __launch_bounds__(kFactorThreads) k_gp_factor_rl(GpDev g, KernelParams k, double noise, double jitter,
                                                              int n) {
  extern __shared__ double A[];  // packed rows [0, n), then c [n], e [n]
  __shared__ double lanes[3][256];
  __shared__ double red[32];
  double* cs = A + even_up(packed(n));
  double* es = cs + n;
  double* colj = es + n;  // column j below the diagonal, contiguous (conflict-free trailing reads)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
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
  // Gram matrix below the diagonal, direct differences (gp.hpp:110), in
  // cta_border_row's argument order
  for (int i = w; i < n; i += nw)
    for (int q = lane; q < i; q += 32)
      A[packed(i) + q] = direct_kernel<NU>(g.train_x + (int64_t)q * g.d, g.train_x + (int64_t)i * g.d, g.d,
                                           k.lengthscale, k.s2);
  const double diag = __dadd_rn(matern<NU>(0.0, k.lengthscale, k.s2), __dadd_rn(noise, jitter));
  __syncthreads();
  const double y0 = n > 0 ? g.y[0] : 0.0;
  double ynext = (threadIdx.x == 0 && n > 0) ? g.y[0] : 0.0;  // thread 0: y[j], loaded a step ahead
  for (int j = 0; j < n; ++j) {
    const double yj = ynext;
    if (threadIdx.x == 0 && j + 1 < n) ynext = g.y[j + 1];
    // row j is final left of the diagonal: its pivot sum and its c / e dot
    // products (cta_ce_row) in one 256-lane tree reduction
    const double* Aj = A + packed(j);
    for (int v = threadIdx.x; v < 256; v += blockDim.x) {
      double sq = 0.0, pc = 0.0, pe = 0.0;
      for (int q = v; q < j; q += 256) {
        sq = __dadd_rn(sq, __dmul_rn(Aj[q], Aj[q]));
        pc = __dadd_rn(pc, __dmul_rn(Aj[q], cs[q]));
        pe = __dadd_rn(pe, __dmul_rn(Aj[q], es[q]));
      }
      lanes[0][v] = sq;
      lanes[1][v] = pc;
      lanes[2][v] = pe;
    }
    double sums[3];
    vsum256<3>(lanes, sums, red);
    const double x = __dadd_rn(diag, -sums[0]);
    if (x <= 0.0) {  // Eigen LLT fails exactly when x <= 0 (a NaN pivot proceeds)
      if (threadIdx.x == 0) {
        g.sc->status = 1;
        g.sc->fail_row = j;
        g.sc->n = 0;
      }
      return;
    }
    const double ljj = sqrt(x), rj = __drcp_rn(ljj);
    for (int q = threadIdx.x; q < j; q += blockDim.x) g.L[packed(j) + q] = Aj[q];  // row j is final
    if (threadIdx.x == 0) {
      A[packed(j) + j] = ljj;
      g.L[packed(j) + j] = ljj;
      const double yr = __dadd_rn(yj, -y0);
      cs[j] = __ddiv_rn(__dadd_rn(yr, -sums[1]), ljj);
      es[j] = __ddiv_rn(__dadd_rn(1.0, -sums[2]), ljj);
      g.c[j] = cs[j];
      g.e[j] = es[j];
    }
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
      const double l = __dmul_rn(A[packed(i) + j], rj);
      A[packed(i) + j] = l;
      colj[i] = l;
    }
    __syncthreads();
    for (int i = j + 2 + w; i < n; i += nw) {
      double* Ai = A + packed(i);
      const double lij = colj[i];
      for (int kk = j + 1 + lane; kk < i; kk += 32) Ai[kk] = __dadd_rn(Ai[kk], -__dmul_rn(colj[kk], lij));
    }
    __syncthreads();
  }
  cta_stats_beta(g, n);
}

template <int NU>
__device__ void gp_append_body(const AppendArgs& a) {
  const GpDev& g = a.g;
  const KernelParams k = a.k;
  const double noise = a.noise;
  const int64_t pos = a.pos;
  const int n0 = a.n0;
  extern __shared__ double smem[];
  __shared__ double red[32];
  const CtaSmem m = cta_smem_layout(smem, g.n_max, n0 + 1, a.staged != 0);
  pdl_begin();
  unsigned long long* tm = g.sc->t;
  if (a.visited_mark && threadIdx.x == 0) a.visited_mark[pos >> 5] |= 1u << (pos & 31);
  append_prologue(g, a.sp, pos, a.x_explicit, a.y_new, n0);
  if (threadIdx.x == 0) tm[0] = gtc_globaltimer();
  if (a.V && pos >= 0) {
    const double* col = a.V + (pos / kTile) * a.tile_stride + pos % kTile;
    if (column_border_row(g, k, noise, col, kTile, n0, m.xs)) return;
    if (threadIdx.x == 0) ++g.sc->exact_rows;
  }
  // exact bordered row: forward substitution over the staged factor
  cta_stage_L(g, n0, m);  // includes __syncthreads
  {
    const double* lp = lp_of(g, m);
    for (int i = threadIdx.x; i < n0; i += blockDim.x) m.rinv[i] = __drcp_rn(lp[packed(i) + i]);
  }  // visible after the Gram-row barrier in cta_border_row
  if (threadIdx.x == 0) tm[1] = gtc_globaltimer();
  const double jitter = g.sc->jitter;
  if (!cta_border_row<NU>(g, k, noise, jitter, n0, m, red, tm)) return;
  if (threadIdx.x == 0) tm[4] = gtc_globaltimer();
  cta_ce_row(g, n0, m, red);
  if (threadIdx.x == 0) tm[5] = gtc_globaltimer();
  cta_stats_beta(g, n0 + 1);
  if (threadIdx.x == 0) tm[6] = gtc_globaltimer();
}

template <int NU>
__global__ void __launch_bounds__(kCtaThreads) k_gp_append(AppendArgs a) {
  gp_append_body<NU>(a);
}

// One CTA per run of a batch (gtc_observe requests gathered across runs).
template <int NU>
__global__ void __launch_bounds__(kCtaThreads) k_gp_append_batch(const AppendArgs* __restrict__ args) {
  const AppendArgs a = args[blockIdx.x];
  if (a.g.L == nullptr) return;  // this run does not append in this batch
  gp_append_body<NU>(a);
}

__global__ void k_gp_truncate(GpDev g, int n) {
  cta_stats_beta(g, n);
}

// ------------------------------------------------------------ V extension

// Coordinates t of candidates j0, j0 + 1 (j0 even): from the compact index
// copy when the space has one (1-byte loads, exact table values), else SoA.
__device__ __forceinline__ double2 coord2(const SpaceDev& sp, int t, int64_t j0) {
  if (sp.cidx) {
    const uchar2 ix = *reinterpret_cast<const uchar2*>(sp.cidx + (int64_t)t * sp.n_pad + j0);
    return make_double2(__ldg(sp.ctab + t * 256 + ix.x), __ldg(sp.ctab + t * 256 + ix.y));
  }
  return *reinterpret_cast<const double2*>(sp.coords + (int64_t)t * sp.n_pad + j0);
}

// Rows in flight per thread and resident CTAs per SM of the single-row pass
// (the HBM stream needs ~150 KB of loads in flight per SM, tools/bw_bench.cu).
#ifndef GTC_PASS_U
#define GTC_PASS_U 6
#endif
#ifndef GTC_PASS_MINB
#define GTC_PASS_MINB 10
#endif
#ifndef GTC_PASS_DB
#define GTC_PASS_DB 0  // double-buffered row groups
#endif

// The final pass's epilogue for one thread's candidate pair (j0, j0 + 1):
// posterior mean and variance (gp.hpp:162-166), the tile's share of the
// variance total over unvisited candidates (strategies.hpp:406-407, fixed
// point), and the tile summary for the selection's pruning.  Block-wide (one
// CTA per tile, kExtendThreads threads).
__device__ __forceinline__ void pass_epilogue(const ExtendArgs& a, int64_t tile, int64_t j0, double b0, double b1,
                                              double q0, double q1) {
  // mean = k*^T alpha = v^T beta;  var = max(s2 - sum v^2, 0)   (gp.hpp:162-166)
  const double var0 = fmax(__dadd_rn(a.s2, -q0), 0.0), var1 = fmax(__dadd_rn(a.s2, -q1), 0.0);
  *reinterpret_cast<double2*>(a.mu + j0) = make_double2(b0, b1);
  *reinterpret_cast<double2*>(a.var + j0) = make_double2(var0, var1);
  if (a.acc || a.tstat) {
    // one reduction for the epilogue's tile quantities:
    //  - this tile's share of the mean posterior variance over the unvisited
    //    candidates (strategies.hpp:406-407), added to the run's fixed-point
    //    total; consumed by the next kernel on the stream (k_select)
    //  - the tile summary (min mean, max/min variance) for tile pruning
    constexpr int kW = kExtendThreads / 32;
    __shared__ double rs[kW], rmn[kW], rvx[kW], rvn[kW], rsm[kW], rva[kW];
    __shared__ long long rc[kW], rpos[kW];
    const bool in0 = j0 < a.sp.n, in1 = j0 + 1 < a.sp.n;
    const uint32_t w = (in0 && a.visited) ? __ldg(a.visited + (j0 >> 5)) : 0xffffffffu;
    const bool u0 = in0 && !((w >> (j0 & 31)) & 1u);
    const bool u1 = in1 && !((w >> ((j0 + 1) & 31)) & 1u);
    double ts = (u0 ? var0 : 0.0) + (u1 ? var1 : 0.0);
    long long tc = (long long)u0 + (long long)u1;
    // bounds over all candidates; seed = unvisited argmin of the mean
    double mn = fmin(in0 ? b0 : CUDART_INF, in1 ? b1 : CUDART_INF);
    double vx = fmax(in0 ? var0 : -CUDART_INF, in1 ? var1 : -CUDART_INF);
    double vn = fmin(in0 ? var0 : CUDART_INF, in1 ? var1 : CUDART_INF);
    double sm_ = u0 ? b0 : CUDART_INF, sv = u0 ? var0 : 0.0;
    long long sp = u0 ? j0 : LLONG_MAX;
    if (u1 && (b1 < sm_ || sp == LLONG_MAX)) {
      sm_ = b1;
      sv = var1;
      sp = j0 + 1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ts += __shfl_xor_sync(0xffffffffu, ts, o);
      tc += __shfl_xor_sync(0xffffffffu, tc, o);
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      vx = fmax(vx, __shfl_xor_sync(0xffffffffu, vx, o));
      vn = fmin(vn, __shfl_xor_sync(0xffffffffu, vn, o));
      const double osm = __shfl_xor_sync(0xffffffffu, sm_, o), osv = __shfl_xor_sync(0xffffffffu, sv, o);
      const long long osp = __shfl_xor_sync(0xffffffffu, sp, o);
      if (osm < sm_ || (osm == sm_ && osp < sp)) {
        sm_ = osm;
        sv = osv;
        sp = osp;
      }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
      rs[wid] = ts;
      rc[wid] = tc;
      rmn[wid] = mn;
      rvx[wid] = vx;
      rvn[wid] = vn;
      rsm[wid] = sm_;
      rva[wid] = sv;
      rpos[wid] = sp;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 1; k < kW; ++k) {  // fixed order
        ts += rs[k];
        tc += rc[k];
        mn = fmin(mn, rmn[k]);
        vx = fmax(vx, rvx[k]);
        vn = fmin(vn, rvn[k]);
        if (rsm[k] < sm_ || (rsm[k] == sm_ && rpos[k] < sp)) {
          sm_ = rsm[k];
          sv = rva[k];
          sp = rpos[k];
        }
      }
      if (a.acc) accum_add(a.acc, ts, tc, a.s2);
#ifdef GTC_SEL_TRACE
      atomicMax(&g_sel_trace[2043][0], gtc_globaltimer());
#endif
      if (a.tstat)
        a.tstat[tile] =
            TileStats{mn, vx >= 0.0 ? vx : -1.0, vn, sm_, sv, sp == LLONG_MAX ? -1 : (int64_t)sp};
    }
  }
}

// Rows [n0, n0+r) of V for every candidate, r <= R, streaming rows [0, n0)
// once.  One CTA per tile of kTile candidates, one double2 column pair per
// thread.  With final_pass the posterior mean/variance are produced too.
template <int R, int NU, int UP = GTC_PASS_U>
__device__ __forceinline__ void extend_body(const ExtendArgs& a_in, int64_t tile_ = -1) {
  ExtendArgs a = a_in;
  const int64_t tile = tile_ >= 0 ? tile_ : (int64_t)blockIdx.x;
  pdl_begin();
  if (blockIdx.x == 0) TRACE_AT(2041, 0);
  // resident loop: only after a valid evaluation; generation flipped by
  // loop_advance.  One thread per CTA reads the loop state and the status
  // word (every CTA reads the same words: one request per CTA, not per warp).
  __shared__ int s_n0, s_gen, s_status;
  __shared__ VarAccum* s_acc;
  if (threadIdx.x == 0) {
    if (a.loop) {
      const LoopDev* lp = a.loop;
      s_n0 = (lp->halt != kLoopRunning || !lp->valid) ? -1 : lp->n0;
      s_gen = lp->gen;
      s_acc = lp->acc;
    }
    s_status = a.check_status ? a.g.sc->status : 0;
  }
  __syncthreads();
  if (a.loop) {
    if (s_n0 < 0) return;
    a.n0 = s_n0;
    a.acc = s_acc + s_gen;
    a.acc_clear = s_acc + (s_gen ^ 1);
  }
  accum_clear(a.acc_clear);  // next generation's accumulator (even when the pass is skipped)
  if (s_status != 0) return;  // bordered row failed: host refactors
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
  if (blockIdx.x == 0) TRACE_AT(2041, 1);
#ifdef GTC_SEL_TRACE
  if (threadIdx.x == 0) atomicMax(&g_sel_trace[2041][2], gtc_globaltimer());  // last CTA through its staging
#endif

  const int64_t j0 = tile * kTile + 2 * threadIdx.x;
  const double2* Vt = reinterpret_cast<const double2*>(a.V + tile * a.tile_stride) + threadIdx.x;
  constexpr int kRowStride = kTile / 2;  // in double2

  double acc0[R], acc1[R];
#pragma unroll
  for (int t = 0; t < R; ++t) acc0[t] = acc1[t] = 0.0;
  double q0 = 0.0, q1 = 0.0, b0 = 0.0, b1 = 0.0;  // sum v^2, sum v*beta

  // U rows in flight; the last partial group is predicated inside the same
  // unrolled body (a scalar remainder loop would serialise its loads)
  constexpr int U = (R == 1) ? UP : 4;
  // rows [i, i + U) into the accumulators, ascending (the reference's order)
  auto consume = [&](const double2 (&v)[U], int i) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i + u >= n0) break;
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
  };
  auto fetch = [&](double2 (&v)[U], int i) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      v[u] = i + u < n0 ? __ldcs(Vt + (int64_t)(i + u) * kRowStride) : make_double2(0.0, 0.0);
  };
  if (GTC_PASS_DB) {
    // two groups in flight: the next group's loads are issued before the
    // current group is consumed, so the stream never drains between groups
    double2 va[U], vb[U];
    fetch(va, 0);
    for (int i = 0; i < n0; i += 2 * U) {
      fetch(vb, i + U);
      consume(va, i);
      fetch(va, i + 2 * U);
      consume(vb, i + U);
    }
  } else {
    for (int i = 0; i < n0; i += U) {
      double2 v[U];
      fetch(v, i);
      consume(v, i);
    }
  }

  // candidate coordinates (SoA) and squared norms, gp.hpp:176-179 expansion
  const int d = a.sp.d;
  double c0n2 = 0.0, c1n2 = 0.0;
  for (int t = 0; t < d; ++t) {
    const double2 c = coord2(a.sp, t, j0);
    c0n2 = __dadd_rn(c0n2, __dmul_rn(c.x, c.x));
    c1n2 = __dadd_rn(c1n2, __dmul_rn(c.y, c.y));
  }
  double vn0[R], vn1[R];
#pragma unroll
  for (int t = 0; t < R; ++t) {
    if (t < r) {
      double dot0 = 0.0, dot1 = 0.0;
      for (int s = 0; s < d; ++s) {
        const double2 c = coord2(a.sp, s, j0);
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
  if (a.final_pass) pass_epilogue(a, tile, j0, b0, b1, q0, q1);
}

// ---- wide streaming rebuild: 32 rows of V per pass (four 8-row panels)
//
// The full forward substitution V = L^-1 K* (gp.hpp:163-164) for the fit,
// refits and predict, with exactly the arithmetic of the 8-row passes
// (k_extend<8>): for row t of panel q
//   acc  = sum_{m < n0 + 8q} L[t][m] v_m    ascending FMA chain: the streamed
//          prefix m < n0, then the pass's earlier panels m in [n0, n0 + 8q)
//   num  = k(x_t, x) - acc;  num -= L[t][s] v_s for s in panel q, s < t;
//   v_t  = num / L[t][t]                     (quot_rn == __ddiv_rn)
// but each pass streams the V prefix ONCE for 32 rows instead of 8: the
// prefix traffic N 8 n^2 / 64 instead of / 16 (5.4 GB instead of 24 GB at
// N = 1M, n = 220), and every loaded V row feeds 64 FMAs per thread (two
// candidates x 32 rows) -- the rebuild becomes FP64-bound rather than
// HBM-bound.  The pass's rows of L are staged transposed in shared memory
// ([m][32]: two rows per 16-byte broadcast load).  The final pass adds the
// posterior (pass_epilogue, the same accumulation order over the rows).
constexpr int kWideRows = 32;
#ifndef GTC_WIDE_U
#define GTC_WIDE_U 4
#endif

__host__ __device__ __forceinline__ size_t wide_smem_doubles(int n0, int d, bool kstar = false) {
  return (size_t)(n0 + kWideRows) * kWideRows + (size_t)(n0 + kWideRows) + (size_t)kWideRows * d + 2 * kWideRows +
         (kstar ? 0 : (size_t)2 * 8 * kExtendThreads);  // + one panel's kernel values [8][threads] double2
}

// Kernel values k(x_t, x) of rows [0, n) for every candidate, written into V
// row t (k_extend_wide then reads them back and overwrites them with v_t):
// the exp / sqrt / division work of the rebuild at full occupancy (8 rows x 2
// candidates per thread), in extend_body's expansion-form order (gp.hpp:176-179).
// DMAX > 0: the candidates' coordinates are decoded once into registers
// (d <= DMAX) instead of once per row -- the kernel is issue-bound (ncu: 84 %
// SM throughput, 1.5e9 warp instructions at n = 220, N = 1M); same
// arithmetic order either way.
constexpr int kKstarRows = 32;  // rows per CTA (the coordinate decode amortised over them)
template <int NU, int DMAX>
__global__ void __launch_bounds__(kExtendThreads) k_kstar(ExtendArgs a, int n) {
  const int d = a.g.d;
  const int64_t tile = blockIdx.x;
  const int64_t j0 = tile * kTile + 2 * threadIdx.x;
  double2 cc[DMAX > 0 ? DMAX : 1];
  double c0n2 = 0.0, c1n2 = 0.0;
  for (int t = 0; t < d; ++t) {
    const double2 c = coord2(a.sp, t, j0);
    if (DMAX > 0) {
#pragma unroll
      for (int q = 0; q < (DMAX > 0 ? DMAX : 1); ++q)
        if (q == t) cc[q] = c;
    }
    c0n2 = __dadd_rn(c0n2, __dmul_rn(c.x, c.x));
    c1n2 = __dadd_rn(c1n2, __dmul_rn(c.y, c.y));
  }
  double2* Vw = reinterpret_cast<double2*>(a.V + tile * a.tile_stride) + threadIdx.x;
  const int t0 = kKstarRows * blockIdx.y, t1 = min(n, t0 + kKstarRows);
  // the CTA's training rows (and squared norms) in shared memory
  __shared__ double xs[kKstarRows * 8 + kKstarRows];
  const bool staged = DMAX > 0 && d <= 8;
  if (staged) {
    for (int idx = threadIdx.x; idx < (t1 - t0) * d; idx += blockDim.x) xs[idx] = a.g.train_x[(int64_t)t0 * d + idx];
    __syncthreads();
    // squared norms from the coordinates (the factor kernels' order, so the
    // same bits as g.train_n2 -- the kernel values do not wait for the factor)
    for (int t = threadIdx.x; t < t1 - t0; t += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < d; ++q) s = __dadd_rn(s, __dmul_rn(xs[t * d + q], xs[t * d + q]));
      xs[kKstarRows * 8 + t] = s;
    }
    __syncthreads();
  }
  const double linv = __drcp_rn(a.lengthscale);
  for (int t = t0; t < t1; ++t) {
    const double* xr = staged ? xs + (t - t0) * d : a.g.train_x + (int64_t)t * d;
    double dot0 = 0.0, dot1 = 0.0;
    if (DMAX > 0) {
#pragma unroll
      for (int q = 0; q < (DMAX > 0 ? DMAX : 1); ++q) {
        if (q >= d) break;
        const double xv = xr[q];
        dot0 = __dadd_rn(dot0, __dmul_rn(xv, cc[q].x));
        dot1 = __dadd_rn(dot1, __dmul_rn(xv, cc[q].y));
      }
    } else {
      for (int q = 0; q < d; ++q) {
        const double2 c = coord2(a.sp, q, j0);
        const double xv = __ldg(xr + q);
        dot0 = __dadd_rn(dot0, __dmul_rn(xv, c.x));
        dot1 = __dadd_rn(dot1, __dmul_rn(xv, c.y));
      }
    }
    double xn2;
    if (staged) {
      xn2 = xs[kKstarRows * 8 + (t - t0)];
    } else {
      xn2 = 0.0;
      for (int q = 0; q < d; ++q) xn2 = __dadd_rn(xn2, __dmul_rn(__ldg(xr + q), __ldg(xr + q)));
    }
    const double d20 = __dadd_rn(__dadd_rn(__dmul_rn(-2.0, dot0), xn2), c0n2);
    const double d21 = __dadd_rn(__dadd_rn(__dmul_rn(-2.0, dot1), xn2), c1n2);
    Vw[(int64_t)t * (kTile / 2)] = make_double2(matern_q<NU>(sqrt(fmax(d20, 0.0)), a.lengthscale, linv, a.s2),
                                                matern_q<NU>(sqrt(fmax(d21, 0.0)), a.lengthscale, linv, a.s2));
  }
}

template <int NU>
__global__ void __launch_bounds__(kExtendThreads, 3) k_extend_wide(ExtendArgs a) {
  extern __shared__ double sm[];
  const int n0 = a.n0, r = a.r, d = a.g.d;
  constexpr int R = kWideRows;
  double* LT = sm;                          // [n0 + R][R]: LT[m * R + t] = L[n0 + t][m] (0 past the row)
  double* bs = LT + (size_t)(n0 + R) * R;   // [n0 + r] beta (final pass)
  double* xn = bs + (n0 + R);               // [R][d] new training coords
  double* xn2 = xn + R * d;                 // [R] their squared norms
  double* rinv = xn2 + R;                   // [R] 1 / L[t][t]
  for (int idx = threadIdx.x; idx < (n0 + R) * R; idx += blockDim.x) {
    const int m = idx / R, t = idx % R;
    LT[idx] = (t < r && m <= n0 + t) ? a.g.L[packed(n0 + t) + m] : 0.0;
  }
  if (a.final_pass)
    for (int q = threadIdx.x; q < n0 + r; q += blockDim.x) bs[q] = a.g.beta[q];
  for (int idx = threadIdx.x; idx < r * d; idx += blockDim.x) xn[idx] = a.g.train_x[(int64_t)n0 * d + idx];
  for (int t = threadIdx.x; t < R; t += blockDim.x) {
    xn2[t] = t < r ? a.g.train_n2[n0 + t] : 0.0;
    rinv[t] = t < r ? __drcp_rn(a.g.L[packed(n0 + t) + n0 + t]) : 1.0;
  }
  __syncthreads();

  const int64_t tile = blockIdx.x;
  const int64_t j0 = tile * kTile + 2 * threadIdx.x;
  const double2* Vt = reinterpret_cast<const double2*>(a.V + tile * a.tile_stride) + threadIdx.x;
  constexpr int kRowStride = kTile / 2;  // in double2
  double acc0[R], acc1[R];
#pragma unroll
  for (int t = 0; t < R; ++t) acc0[t] = acc1[t] = 0.0;
  double q0 = 0.0, q1 = 0.0, b0 = 0.0, b1 = 0.0;
  constexpr int U = GTC_WIDE_U;
  for (int i = 0; i < n0; i += U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      v[u] = i + u < n0 ? __ldcs(Vt + (int64_t)(i + u) * kRowStride) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i + u >= n0) break;
      const double2* lt = reinterpret_cast<const double2*>(LT + (size_t)(i + u) * R);
#pragma unroll
      for (int t2 = 0; t2 < R / 2; ++t2) {
        const double2 l = lt[t2];
        acc0[2 * t2] = fma(l.x, v[u].x, acc0[2 * t2]);
        acc1[2 * t2] = fma(l.x, v[u].y, acc1[2 * t2]);
        acc0[2 * t2 + 1] = fma(l.y, v[u].x, acc0[2 * t2 + 1]);
        acc1[2 * t2 + 1] = fma(l.y, v[u].y, acc1[2 * t2 + 1]);
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
  // candidate coordinates and squared norms (extend_body's order)
  double c0n2 = 0.0, c1n2 = 0.0;
  for (int t = 0; t < d; ++t) {
    const double2 c = coord2(a.sp, t, j0);
    c0n2 = __dadd_rn(c0n2, __dmul_rn(c.x, c.x));
    c1n2 = __dadd_rn(c1n2, __dmul_rn(c.y, c.y));
  }
  double2* Vw = reinterpret_cast<double2*>(a.V + tile * a.tile_stride) + threadIdx.x;
  // kernel values of each panel's rows first (from k_kstar's V rows, or
  // evaluated here into this thread's shared slots: independent evaluations,
  // so the exp / sqrt / division chains overlap instead of sitting on the
  // triangle's dependency chain)
  double2* kv = reinterpret_cast<double2*>(rinv + R) + threadIdx.x;  // [8][kExtendThreads] double2
  // the pass's rows, panel by panel; acc0/acc1[t] become v once row t is done
#pragma unroll
  for (int pq = 0; pq < R / 8; ++pq) {
  for (int t = 8 * pq; !a.kstar && t < min(r, 8 * pq + 8); ++t) {
    double dot0 = 0.0, dot1 = 0.0;
    for (int q = 0; q < d; ++q) {
      const double2 c = coord2(a.sp, q, j0);
      const double xv = xn[t * d + q];
      dot0 = __dadd_rn(dot0, __dmul_rn(xv, c.x));
      dot1 = __dadd_rn(dot1, __dmul_rn(xv, c.y));
    }
    const double d20 = __dadd_rn(__dadd_rn(__dmul_rn(-2.0, dot0), xn2[t]), c0n2);
    const double d21 = __dadd_rn(__dadd_rn(__dmul_rn(-2.0, dot1), xn2[t]), c1n2);
    kv[(t - 8 * pq) * kExtendThreads] = make_double2(matern<NU>(sqrt(fmax(d20, 0.0)), a.lengthscale, a.s2),
                                                     matern<NU>(sqrt(fmax(d21, 0.0)), a.lengthscale, a.s2));
  }
#pragma unroll
    for (int t = 8 * pq; t < 8 * pq + 8; ++t) {
      if (t >= r) break;
      // the FMA chain continued over the earlier panels of this pass (ascending)
#pragma unroll
      for (int s = 0; s < 8 * pq; ++s) {
        const double l = LT[(size_t)(n0 + s) * R + t];
        acc0[t] = fma(l, acc0[s], acc0[t]);
        acc1[t] = fma(l, acc1[s], acc1[t]);
      }
      const double2 kk = a.kstar ? Vw[(int64_t)(n0 + t) * kRowStride] : kv[(t - 8 * pq) * kExtendThreads];
      double num0 = __dadd_rn(kk.x, -acc0[t]);
      double num1 = __dadd_rn(kk.y, -acc1[t]);
#pragma unroll
      for (int s = 8 * pq; s < t; ++s) {
        const double l = LT[(size_t)(n0 + s) * R + t];
        num0 = __dadd_rn(num0, -__dmul_rn(l, acc0[s]));
        num1 = __dadd_rn(num1, -__dmul_rn(l, acc1[s]));
      }
      const double diag = LT[(size_t)(n0 + t) * R + t];
      acc0[t] = quot_rn(num0, diag, rinv[t]);
      acc1[t] = quot_rn(num1, diag, rinv[t]);
      Vw[(int64_t)(n0 + t) * kRowStride] = make_double2(acc0[t], acc1[t]);
      if (a.final_pass) {
        const double bb = bs[n0 + t];
        q0 = fma(acc0[t], acc0[t], q0);
        q1 = fma(acc1[t], acc1[t], q1);
        b0 = fma(acc0[t], bb, b0);
        b1 = fma(acc1[t], bb, b1);
      }
    }
  }
  if (a.final_pass) pass_epilogue(a, tile, j0, b0, b1, q0, q1);
}

// ---- wide rebuild on the FP64 tensor cores: 32 rows per pass, DMMA contraction
//
// The 32-row passes of k_extend_wide with the prefix contraction
//   acc[t][x] = sum_{m < n0} L[n0 + t][m] v_m(x)
// as FP64 mma.sync m8n8k4 (DMMA): a warp owns 8 candidates and the four
// 8-row panels of the pass (four 8x8 accumulator fragments); each k-step
// loads ONE B fragment (4 V rows x 8 candidates, streamed from HBM) and
// reuses it for the four panels' A fragments (L rows staged in shared
// memory).  A chain of DMMAs is the ascending FMA chain
// (tools/dmma_order.cu), so the prefix part, the continuation over the
// pass's earlier panels (DMMA again, B from the panels' v in shared memory)
// and the panel triangles (shuffle broadcast, quot_rn == __ddiv_rn) are the
// 8-row passes' arithmetic bit for bit.  Four accumulator fragments are 8
// doubles per thread instead of 64, so 24 warps per SM keep 8 k-steps of the
// stream in flight.  The kernel values come from k_kstar; the posterior from
// a following r = 0 pass.
constexpr int kWmWarps = 8;  // warps (8 candidates each) per CTA
constexpr int kWmU = 8;      // k-steps of B fragments in flight per warp

__host__ __device__ __forceinline__ int wm_ld(int n0) { return ((n0 + kWideRows + 15) / 16) * 16 + 4; }
__host__ __device__ __forceinline__ size_t wm_smem_doubles(int n0) {
  return (size_t)kWideRows * wm_ld(n0) + kWideRows + (size_t)kWmWarps * 4 * 64;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kWmWarps * 32, 3) k_extend_wide_mma(ExtendArgs a) {
  extern __shared__ double sm[];
  constexpr int R = kWideRows;
  const int n0 = a.n0, r = a.r, ld = wm_ld(n0);
  double* Ls = sm;             // [R][ld]: Ls[t * ld + m] = L[n0 + t][m] for m <= n0 + t, rows t < r; else 0
  double* rinvs = Ls + R * ld;  // [R] 1 / L[n0 + t][n0 + t]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* vbuf = rinvs + R + (size_t)w * 4 * 64;  // [4 panels][8 rows][8 candidates] this warp's v
  for (int idx = threadIdx.x; idx < R * ld; idx += blockDim.x) {
    const int t = idx / ld, m = idx % ld;
    Ls[idx] = (t < r && m <= n0 + t) ? a.g.L[packed(n0 + t) + m] : 0.0;
  }
  for (int t = threadIdx.x; t < R; t += blockDim.x) rinvs[t] = t < r ? __drcp_rn(a.g.L[packed(n0 + t) + n0 + t]) : 1.0;
  __syncthreads();
  const int row = lane >> 2, kq = lane & 3, col = 2 * kq;
  const int64_t c0 = ((int64_t)blockIdx.x * kWmWarps + w) * 8;  // this warp's first candidate
  if (c0 >= a.sp.n_pad) return;
  double* Vt = a.V + (c0 / kTile) * a.tile_stride + c0 % kTile;  // row m of the warp's candidates at Vt + m * kTile
  double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  // ---- the prefix: rows m < n0 (n0 is a multiple of 32), B streamed, kWmU k-steps in flight
  const double* Bp = Vt + (int64_t)kq * kTile + row;  // B fragment of k-step m0: V[m0 + kq][row]
  for (int m0 = 0; m0 < n0; m0 += 4 * kWmU) {
    double bv[kWmU];
#pragma unroll
    for (int u = 0; u < kWmU; ++u) bv[u] = m0 + 4 * u < n0 ? __ldcs(Bp + (int64_t)(m0 + 4 * u) * kTile) : 0.0;
#pragma unroll
    for (int u = 0; u < kWmU; ++u) {
      if (m0 + 4 * u >= n0) break;
      const double* Ap = Ls + row * ld + m0 + 4 * u + kq;
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(d[i], Ap[8 * i * ld], bv[u]);
    }
  }
  // ---- the pass's four panels
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = 8 * i + row;  // this thread's D row
    const bool live = t < r;
    // the FMA chain continued over the earlier panels (DMMA, B from their v)
#pragma unroll
    for (int j = 0; j < i; ++j) {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const double av = Ls[t * ld + n0 + 8 * j + 4 * kk + kq];
        const double bv = vbuf[j * 64 + (4 * kk + kq) * 8 + row];
        dmma(d[i], av, bv);
      }
    }
    // kernel values (k_kstar wrote them into these V rows)
    double2 kk2 = make_double2(0.0, 0.0);
    if (live) kk2 = __ldcg(reinterpret_cast<const double2*>(Vt + (int64_t)(n0 + t) * kTile + col));
    double num0 = __dadd_rn(kk2.x, -d[i][0]), num1 = __dadd_rn(kk2.y, -d[i][1]);
    // the panel triangle (k_extend<8>'s order), row s on lanes 4s .. 4s + 3
    const double diag = live ? Ls[t * ld + n0 + t] : 1.0, rinv = rinvs[t];
    double v0 = 0.0, v1 = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      if (8 * i + s >= r) break;
      const double q0 = quot_rn(num0, diag, rinv), q1 = quot_rn(num1, diag, rinv);
      if (row == s) {
        v0 = q0;
        v1 = q1;
      }
      const double b0 = __shfl_sync(0xffffffffu, q0, s * 4 + kq);
      const double b1 = __shfl_sync(0xffffffffu, q1, s * 4 + kq);
      const double l = Ls[t * ld + n0 + 8 * i + s];
      if (row > s) {
        num0 = __dadd_rn(num0, -__dmul_rn(l, b0));
        num1 = __dadd_rn(num1, -__dmul_rn(l, b1));
      }
    }
    if (!live) v0 = v1 = 0.0;  // (rows past the model: zero B entries for the later panels)
    *reinterpret_cast<double2*>(vbuf + i * 64 + row * 8 + col) = make_double2(v0, v1);
    if (live) *reinterpret_cast<double2*>(Vt + (int64_t)(n0 + t) * kTile + col) = make_double2(v0, v1);
    __syncwarp();
  }
}

// ---- persistent 64-row DMMA passes (GTC_REBUILD=pmma, mode 4)
//
// The same 8-row panel arithmetic as k_extend_wide_mma, regrouped so the
// FP64 tensor cores are fed from half the stream with no per-CTA staging in
// the steady state:
//  * 64 rows (eight 8-row panels) per pass: every streamed B fragment feeds
//    eight panels' A fragments (2.9 instead of 5.4 GB of prefix reads at
//    n = 220), four passes instead of seven;
//  * a warp owns 16 candidates as two interleaved 8-candidate groups (even /
//    odd positions): one 16-byte load per lane and k-step gives both groups'
//    B fragments from full 128-byte lines, and each A fragment feeds two DMMAs;
//  * one persistent CTA per SM stages the pass's rows of L once and loops
//    over candidate groups (no per-CTA L staging on the critical path);
//  * the continuation over the pass's earlier panels is right-looking: once
//    panel j is solved its v (re-laid out to the B fragment layout through
//    the warp's shared buffer) updates panels i > j at once, so row t of
//    panel i still sees the ascending chain prefix, panel 0, ..., panel i-1
//    -- bit for bit the FMA chain of k_extend<8> (tools/dmma_order.cu).
constexpr int kPmRows = 64;
constexpr int kPmWarps = 16;
#ifndef GTC_PM_RING
#define GTC_PM_RING 8
#endif
constexpr int kPmRingSteps = GTC_PM_RING;  // k-steps of B in each warp's shared ring (0: register path)
#ifndef GTC_PM_U
#define GTC_PM_U 4
#endif

// ld = 8 (mod 16) doubles: the paired A loads below are conflict-free per
// 8-lane phase.  Within every 8-column block the columns are stored paired
// (column m0 + q at m0 + 2q, m0 + 4 + q at m0 + 2q + 1), so one 16-byte load
// gives a lane its A elements of two consecutive k-steps.
__host__ __device__ __forceinline__ int pm_ld(int n0) { return ((n0 + kPmRows + 15) / 16) * 16 + 8; }
__host__ __device__ __forceinline__ int pm_perm(int m) { return (m & ~7) | ((m & 3) << 1) | ((m >> 2) & 1); }
__host__ __device__ __forceinline__ size_t pm_smem_doubles(int n0, bool ring) {
  // + the panels' diagonal blocks [8][8][8] + per-warp triangle buffers (+ B rings)
  return (size_t)kPmRows * pm_ld(n0) + kPmRows + 8 * 64 + (size_t)kPmWarps * 128 +
         (ring ? (size_t)kPmWarps * kPmRingSteps * 64 : 0);
}

__device__ __forceinline__ void pm_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void pm_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void pm_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(kPmWarps * 32, 1) k_extend_pm(ExtendArgs a, int* __restrict__ next_group, int use_ring) {
  extern __shared__ double sm[];
  constexpr int R = kPmRows, U = GTC_PM_U;
  const int n0 = a.n0, r = a.r, ld = pm_ld(n0);
  const int P = (r + 7) / 8;    // live panels of this pass
  double* Ls = sm;              // [R][ld]: Ls[t * ld + m] = L[n0 + t][m] for m <= n0 + t, rows t < r; else 0
  double* rinvs = Ls + R * ld;  // [R] 1 / L[n0 + t][n0 + t]
  double* Lb = rinvs + R;       // [8 panels][8][8]: Lb[j * 64 + t * 8 + s] = L[n0 + 8j + t][n0 + 8j + s] (s <= t)
  for (int idx = threadIdx.x; idx < R * ld; idx += blockDim.x) {
    const int t = idx / ld, m = idx % ld;  // Ls[t * ld + pm_perm(m)] = L[n0 + t][m]
    Ls[t * ld + pm_perm(m)] = (t < r && m <= n0 + t) ? a.g.L[packed(n0 + t) + m] : 0.0;
  }
  for (int t = threadIdx.x; t < R; t += blockDim.x) rinvs[t] = t < r ? __drcp_rn(a.g.L[packed(n0 + t) + n0 + t]) : 1.0;
  for (int idx = threadIdx.x; idx < 8 * 64; idx += blockDim.x) {
    const int j = idx >> 6, t = (idx >> 3) & 7, q = idx & 7, tr = 8 * j + t;
    Lb[idx] = (tr < r && q <= t) ? a.g.L[packed(n0 + tr) + n0 + 8 * j + q] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int row = lane >> 2, kq = lane & 3;
  const int64_t groups = a.sp.n_pad / 16;
  // groups are handed out dynamically (one atomic per group and warp): a
  // CTA that starts late on a busy SM does not hold the whole pass back
  for (;;) {
    int64_t grp = 0;
    if (lane == 0) grp = atomicAdd(next_group, 1);
    grp = __shfl_sync(0xffffffffu, grp, 0);
    if (grp >= groups) break;
    const int64_t c0 = grp * 16;
    double* Vt = a.V + (c0 / kTile) * a.tile_stride + c0 % kTile;  // row m of the group at Vt + m * kTile
    // d[i][g][c]: panel i, group g (candidates c0 + 2n + g), accumulator column c
    double d[8][2][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i][0][0] = d[i][0][1] = d[i][1][0] = d[i][1][1] = 0.0;
    // the pass's kernel-value rows into L2 now (read after the prefix)
    for (int t = lane; t < r; t += 32)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(Vt + (int64_t)(n0 + t) * kTile));
    // ---- the prefix rows m < n0, B fragments streamed (lane: V[m + kq][c0 + 2 row + {0, 1}])
    const double2* Bp = reinterpret_cast<const double2*>(Vt + (int64_t)kq * kTile) + row;
    static_assert(U % 2 == 0, "k-steps are consumed in pairs");
#if GTC_PM_RING
    // B fragments through a per-warp shared ring filled by cp.async: S
    // k-steps in flight per warp without holding them in registers
    if (use_ring) {
      constexpr int S = GTC_PM_RING;
      static_assert(S % 2 == 0 && S >= 4, "ring of k-step pairs");
      double2* ring = reinterpret_cast<double2*>(Lb + 8 * 64 + kPmWarps * 128) + (size_t)w * S * 32 + lane;
      const int ksteps = n0 / 4;
#pragma unroll
      for (int q = 0; q < S; ++q) {
        if (q < ksteps) pm_cp16(ring + q * 32, Bp + (int64_t)(4 * q) * (kTile / 2));
        pm_commit();
      }
      for (int ks = 0; ks < ksteps; ks += 2) {
        pm_wait<S - 2>();  // k-steps ks, ks + 1 landed
        const int slot = ks % S;
        const double2 b0 = ring[slot * 32], b1 = ring[(slot + 1) * 32];
        const double* Ap = Ls + row * ld + 4 * ks + 2 * kq;  // (k-steps ks and ks + 1)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i >= P) break;
          const double2 av = *reinterpret_cast<const double2*>(Ap + 8 * i * ld);
          dmma(d[i][0], av.x, b0.x);
          dmma(d[i][1], av.x, b0.y);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i >= P) break;
          const double2 av = *reinterpret_cast<const double2*>(Ap + 8 * i * ld);
          dmma(d[i][0], av.y, b1.x);
          dmma(d[i][1], av.y, b1.y);
        }
        // refill the two slots (after their values were consumed by the DMMAs above)
        if (ks + S < ksteps) pm_cp16(ring + slot * 32, Bp + (int64_t)(4 * (ks + S)) * (kTile / 2));
        pm_commit();
        if (ks + S + 1 < ksteps) pm_cp16(ring + (slot + 1) * 32, Bp + (int64_t)(4 * (ks + S + 1)) * (kTile / 2));
        pm_commit();
      }
      pm_wait<0>();
    } else
#endif
    for (int m0 = 0; m0 < n0; m0 += 4 * U) {  // (n0 is a multiple of 64)
      double2 bv[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        bv[u] = m0 + 4 * u < n0 ? __ldcs(Bp + (int64_t)(m0 + 4 * u) * (kTile / 2)) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < U; u += 2) {
        if (m0 + 4 * u >= n0) break;
        const double* Ap = Ls + row * ld + m0 + 4 * u + 2 * kq;  // (k-steps m0 + 4u and m0 + 4u + 4)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i >= P) break;
          const double2 av = *reinterpret_cast<const double2*>(Ap + 8 * i * ld);
          dmma(d[i][0], av.x, bv[u].x);
          dmma(d[i][1], av.x, bv[u].y);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i >= P) break;
          const double2 av = *reinterpret_cast<const double2*>(Ap + 8 * i * ld);
          dmma(d[i][0], av.y, bv[u + 1].x);
          dmma(d[i][1], av.y, bv[u + 1].y);
        }
      }
    }
    // ---- the pass's panels, each solved then applied to the later ones.
    // The triangle runs one candidate per lane (lanes c and c + 16 both own
    // candidate c0 + c): the accumulators go through this warp's shared
    // buffer tb[8 rows][16 candidates], the candidate's 8 rows are solved in
    // registers, v goes back through tb to the B fragment layout.
    double* tb = Lb + 8 * 64 + w * 128;
    const int cl = lane & 15;
    // kernel values of the panel's rows for this lane's candidate (k_kstar),
    // the next panel's in flight while this one is solved
    double kvn[8];
#pragma unroll
    for (int tt = 0; tt < 8; ++tt) kvn[tt] = tt < r ? __ldcg(Vt + (int64_t)(n0 + tt) * kTile + cl) : 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j >= P) break;
      const int rows = min(8, r - 8 * j);
      double kv[8];
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        kv[tt] = kvn[tt];
        kvn[tt] = 8 * (j + 1) + tt < r ? __ldcg(Vt + (int64_t)(n0 + 8 * (j + 1) + tt) * kTile + cl) : 0.0;
      }
      // accumulators -> tb: lane (row, kq) holds candidates 4 kq + (g0 c0, g1 c0, g0 c1, g1 c1)
      __syncwarp();
      reinterpret_cast<double2*>(tb + row * 16 + 4 * kq)[0] = make_double2(d[j][0][0], d[j][1][0]);
      reinterpret_cast<double2*>(tb + row * 16 + 4 * kq)[1] = make_double2(d[j][0][1], d[j][1][1]);
      __syncwarp();
      // the panel triangle (k_extend<8>'s order): num = k - acc, then
      // num -= l_ts v_s for s < t ascending (separately rounded), v = num / L_tt
      const double* Lp = Lb + j * 64;  // Lp[tt * 8 + s] = L[n0 + 8j + tt][n0 + 8j + s]
      double v[8];
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        v[tt] = 0.0;
        if (tt < rows) {
          double num = __dadd_rn(kv[tt], -tb[tt * 16 + cl]);
#pragma unroll
          for (int s = 0; s < tt; ++s) num = __dadd_rn(num, -__dmul_rn(Lp[tt * 8 + s], v[s]));
          v[tt] = quot_rn_c(num, Lp[tt * 8 + tt], rinvs[8 * j + tt]);
        }
      }
      __syncwarp();
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        if (lane < 16) tb[tt * 16 + cl] = v[tt];  // (0 for rows past the model: zero B entries)
        if (lane < 16 && tt < rows) Vt[(int64_t)(n0 + 8 * j + tt) * kTile + cl] = v[tt];
      }
      __syncwarp();
      // panel j's v as B fragments (k-step kk: rows 8j + 4kk + kq; group g column row = candidate 2 row + g)
      if (j + 1 < P) {
        const double2 b0 = *reinterpret_cast<const double2*>(tb + kq * 16 + 2 * row);
        const double2 b1 = *reinterpret_cast<const double2*>(tb + (4 + kq) * 16 + 2 * row);
#pragma unroll
        for (int i = j + 1; i < 8; ++i) {
          if (i >= P) break;
          const double2 av = *reinterpret_cast<const double2*>(Ls + (8 * i + row) * ld + n0 + 8 * j + 2 * kq);
          dmma(d[i][0], av.x, b0.x);
          dmma(d[i][1], av.x, b0.y);
          dmma(d[i][0], av.y, b1.x);
          dmma(d[i][1], av.y, b1.y);
        }
      }
    }
  }
}

template <int R, int NU>
__global__ void __launch_bounds__(kExtendThreads, R == 1 ? GTC_PASS_MINB : 4) k_extend(ExtendArgs a) {
  extend_body<R, NU>(a);
}

// Small spaces (fewer tiles than ~4 per SM): too few CTAs to keep enough V
// loads in flight, so each thread keeps kDeepRows rows in flight instead
// (same operations in the same order, only deeper load pipelining).
#ifndef GTC_PASS_U_DEEP
#define GTC_PASS_U_DEEP 16
#endif
template <int NU>
__global__ void __launch_bounds__(kExtendThreads, 4) k_extend_deep(ExtendArgs a) {
  extend_body<1, NU, GTC_PASS_U_DEEP>(a);
}
static bool deep_pass(int64_t tiles);

// Runs of a batch on the y axis (same space, hence the same tiles).
template <int NU>
__global__ void __launch_bounds__(kExtendThreads, GTC_PASS_MINB) k_extend_batch(const ExtendArgs* __restrict__ args) {
  const ExtendArgs a = args[blockIdx.y];
  if (a.V == nullptr) return;  // this run does not append in this batch
  extend_body<1, NU>(a);
}

// Prior (n == 0): mean 0, variance = output variance (gp.hpp:155-158).
__global__ void k_prior(double* mu, double* var, int64_t n, double s2, TileStats* tstat) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    mu[j] = 0.0;
    var[j] = s2;
  }
  if (tstat)
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n / kTile;
         t += (int64_t)gridDim.x * blockDim.x)
      tstat[t] = TileStats{0.0, s2, s2, 0.0, s2, t * kTile};
}

// Marks (or unmarks) one candidate; with `acc`, moves its variance out of (or
// back into) the run's variance total.  The caller guarantees the bit flips.
__device__ __forceinline__ void mark_update(uint32_t* visited, int64_t pos, int set, VarAccum* acc,
                                            const double* var, double s2) {
  if (set)
    atomicOr(visited + (pos >> 5), 1u << (pos & 31));
  else
    atomicAnd(visited + (pos >> 5), ~(1u << (pos & 31)));
  if (acc) accum_add_one(acc, var[pos], set ? -1 : 1, s2);
}

__global__ void k_mark_batch(const MarkDesc* __restrict__ m, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) mark_update(m[i].visited, m[i].pos, 1, m[i].acc, m[i].var, m[i].s2);
}

__global__ void k_mark(uint32_t* visited, int64_t pos, int set, VarAccum* acc, const double* var, double s2) {
  mark_update(visited, pos, set, acc, var, s2);
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
  // fixed-order sum of the block partials (gridDim.x <= 1184)
  s = 0.0;
  c = 0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    s += __ldcg(partial_sum + b);
    c += __ldcg(reinterpret_cast<const long long*>(partial_cnt) + b);
  }
  s = block_sum(s, red);
  c = block_sum_ll(c, redl);
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
  LoopDev* loop;  // resident loop: advanced by the last block (loop_advance)
  const double* pf_table;  // SelectParams::pf_* (L2 warm-up of the winners' table entries / V columns)
  const double* pf_V;
  int64_t pf_tile_stride;
  int32_t pf_rows;
  const double* pf_c;      // SelectParams::pf_gp (the fused append's c, e, y inputs)
  const double* pf_e;
  const double* pf_y;
  SelectDev* host_sel;     // SelectParams::host_* (direct read-back into pinned host memory)
  GpScalars* host_sc;
  uint32_t* host_seq;
  uint32_t seq;
  const GpScalars* sc_src;
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

// Block reduction of the per-thread (best per AF, first eligible + whether
// its keys were finite, count) with one barrier, then the last-block merge
// into the result record.  A finite key implies a finite (non-NaN) score, so
// the first-candidate rule (portfolio.hpp:52: the first eligible candidate is
// taken unconditionally; if its score is NaN nothing beats it) needs an exact
// score only when the global first candidate had non-finite inputs.
struct SelPart {
  Best b[3];
  int64_t first;
  int finite;
  long long cnt;
};

template <uint32_t MASK>
__device__ __forceinline__ SelPart sel_merge(SelPart x, const SelPart& y) {
#pragma unroll
  for (int af = 0; af < 3; ++af)
    if (MASK & (1u << af)) x.b[af] = better(x.b[af], y.b[af]);
  if (y.first < x.first) {
    x.first = y.first;
    x.finite = y.finite;
  }
  x.cnt += y.cnt;
  return x;
}

template <uint32_t MASK>
__device__ __forceinline__ SelPart sel_warp_reduce(SelPart v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    SelPart w;
#pragma unroll
    for (int af = 0; af < 3; ++af) {
      if (!(MASK & (1u << af))) continue;
      w.b[af].s = __shfl_xor_sync(0xffffffffu, v.b[af].s, o);
      w.b[af].p = __shfl_xor_sync(0xffffffffu, v.b[af].p, o);
    }
    w.first = __shfl_xor_sync(0xffffffffu, v.first, o);
    w.finite = __shfl_xor_sync(0xffffffffu, v.finite, o);
    w.cnt = __shfl_xor_sync(0xffffffffu, v.cnt, o);
    v = sel_merge<MASK>(v, w);
  }
  return v;
}

// Resident loop step, run by the selection's last thread once the selection
// is final: its pick is evaluated from the value table and applied to the
// loop state -- the host bookkeeping of gtc_observe (visited mark, candidate
// count, first eligible position, f_best; RunContext::evaluate,
// strategies.hpp:159-232) done on the device.
// Portfolio::next_in_rotation (portfolio.hpp:182-189).
__device__ int port_next(PortDev& P) {
  for (int step = 0; step < 3; ++step) {
    const int a = (int)(P.cursor % 3);
    ++P.cursor;
    if (P.active[a]) return a;
  }
  return -1;
}

// Portfolio::suggest (portfolio.hpp:130-134, suggest_multi :191-218 with
// resolve_duplicates :222-236, suggest_advanced :238-256; the pending set
// is always empty inside run_bo) on the selection's per-AF argmaxes.
__device__ int64_t port_suggest(PortDev& P, const SelectDev* sel, int* by) {
  if (P.mode == 2) {
    const int c = port_next(P);
    *by = c;
    P.last_sug[c] = sel->position[c];
    return sel->position[c];
  }
  int64_t pick[3];
  for (int a = 0; a < 3; ++a) {
    pick[a] = sel->position[a];
    if (P.active[a]) P.last_sug[a] = pick[a];
  }
  const int c = port_next(P);
  *by = c;
  const int64_t chosen = pick[c];
  bool conflict[3] = {false, false, false};
  bool any = false;
  for (int a = 0; a < 3; ++a)
    if (P.active[a] && a != c && P.last_sug[a] == chosen) conflict[a] = any = true;
  if (any) {
    ++P.duplicates[c];
    for (int a = 0; a < 3; ++a)
      if (conflict[a]) ++P.duplicates[a];
    conflict[c] = true;
    bool over = false;
    for (int a = 0; a < 3; ++a) over |= conflict[a] && P.duplicates[a] > P.skip_threshold;
    if (over) {  // keep the lowest discounted observation score (earliest on ties)
      int keep = -1;
      for (int a = 0; a < 3; ++a)
        if (P.active[a] && conflict[a] && (keep < 0 || P.dos[a] < P.dos[keep])) keep = a;
      for (int a = 0; a < 3; ++a)
        if (conflict[a]) {
          P.duplicates[a] = 0;
          if (a != keep) P.active[a] = 0;
        }
    }
  }
  return chosen;
}

// Portfolio::update_bands (portfolio.hpp:259-299).
__device__ void port_update_bands(PortDev& P, int p) {
  if (!P.active[p]) return;
  double mean = 0.0;
  int n = 0;
  for (int a = 0; a < 3; ++a)
    if (P.active[a]) {
      mean = __dadd_rn(mean, P.dos[a]);
      ++n;
    }
  mean = __ddiv_rn(mean, (double)n);
  if (P.dos[p] > __dmul_rn(__dadd_rn(1.0, P.rho), mean))
    ++P.above[p];
  else if (P.dos[p] < __dmul_rn(__dadd_rn(1.0, -P.rho), mean))
    ++P.below[p];
  if (P.below[p] >= P.skip_threshold && n > 1) {
    for (int a = 0; a < 3; ++a) {
      if (a != p) P.active[a] = 0;
      P.above[a] = 0;
      P.below[a] = 0;
    }
    return;
  }
  if (P.above[p] >= P.skip_threshold && n > 1) {
    P.active[p] = 0;
    P.above[p] = 0;
    P.below[p] = 0;
    for (int a = 0; a < 3; ++a)
      if (P.active[a]) {
        P.above[a] = 0;
        P.below[a] = 0;
      }
  }
}

// Portfolio::record (portfolio.hpp:140-150) of an already resolved observed
// value (an invalid result's median is the caller's).
__device__ void port_record(PortDev& P, int by, double observed) {
  P.dos[by] = __dadd_rn(__dmul_rn(P.dos[by], P.discount), observed);
  if (P.mode == 2) port_update_bands(P, by);
}

// This shard's local index of global position `pos` (-1: another shard's);
// without sharding offset = 0 and every position is local.
__device__ __forceinline__ int64_t shard_local(const LoopDev* L, int64_t pos) {
  const int64_t p = pos - L->offset;
  return (p >= 0 && p < L->n_space) ? p : -1;
}

__device__ void loop_advance(LoopDev* L, const SelectDev* sel) {
  if (sel->n_candidates <= 0) {
    L->halt = kLoopNoCandidates;
    return;
  }
  PortDev& P = L->port;
  int by = L->af;
  const int64_t pos = P.mode != 0 ? port_suggest(P, sel, &by) : sel->position[L->af];
  const double y = L->table[pos];
  const int valid = y == y;
  if (valid && !L->hold && L->n >= L->n_max) {
    L->halt = kLoopCapacity;
    return;
  }
  if (P.mode != 0) {
    // Portfolio::record (portfolio.hpp:140-150): invalid -> median of the valid observations
    double observed = y;
    if (!valid) {  // (n_sorted >= 1: the loop starts from a fitted model of the valid observations)
      const int m = L->n_sorted;
      observed = (m & 1) ? L->sorted_y[m / 2]
                         : __dmul_rn(0.5, __dadd_rn(L->sorted_y[m / 2 - 1], L->sorted_y[m / 2]));
    }
    port_record(P, by, observed);
    if (valid) {  // keep the valid observations sorted (insertion)
      int i = L->n_sorted++;
      while (i > 0 && L->sorted_y[i - 1] > y) {
        L->sorted_y[i] = L->sorted_y[i - 1];
        --i;
      }
      L->sorted_y[i] = y;
    }
  }
  L->rec[L->step] = StepRec{pos, y, sel->lambda, valid, sel->cv_fallback, by, 0};
  ++L->step;
  L->pos = pos;
  L->y = y;
  L->valid = valid;
  const int64_t lpos = shard_local(L, pos);  // visited / count / first / acc are the shard's
  if (valid) {
    if (L->hold) {  // steady state: replace the observation at row hold_n0
      const int64_t prev = L->hold_prev >= 0 ? shard_local(L, L->hold_prev) : -1;
      if (prev >= 0) {
        atomicAnd(L->visited + (prev >> 5), ~(1u << (prev & 31)));  // (no return value: a reduction, no round trip)
        ++L->count;
        if (L->first < 0 || prev < L->first) L->first = prev;
      }
      L->hold_prev = pos;
      L->n0 = L->hold_n0;
      L->n = L->hold_n0 + 1;
      L->f_best = y < L->f_base ? y : L->f_base;
    } else {
      L->n0 = L->n;
      ++L->n;
      if (y < L->f_best) L->f_best = y;
    }
    L->gen ^= 1;  // the pass produces the next generation
    if (lpos >= 0) atomicOr(L->visited + (lpos >> 5), 1u << (lpos & 31));
  } else if (lpos >= 0) {
    // no refit: the variance total loses this candidate in O(1)
    mark_update(L->visited, lpos, 1, L->acc + L->gen, L->var, L->s2);
  }
  if (lpos < 0) return;
  --L->count;
  if (lpos == L->first) {  // next unvisited position (first only moves forward within a run)
    const int64_t n = L->n_space, nw = (n + 31) >> 5;
    int64_t found = -1;
    for (int64_t w = lpos >> 5; w < nw; ++w) {
      uint32_t fb = ~L->visited[w];
      if (w == nw - 1 && (n & 31)) fb &= (1u << (n & 31)) - 1u;
      if (fb) {
        found = (w << 5) + (__ffs(fb) - 1);
        break;
      }
    }
    L->first = found;
  }
}

// The device portfolio driven by an explicit script (gtc_portfolio_trace):
// the same port_suggest / port_record the resident loop runs, on given
// per-function argmaxes and observed values (portfolio parity tests).
__global__ void k_portfolio_trace(PortDev P, const PortOp* ops, int n, PortState* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int i = 0; i < n; ++i) {
    PortState& o = out[i];
    o.position = -1;
    o.by = -1;
    if (ops[i].kind == 0) {
      SelectDev sel{};
      for (int a = 0; a < 3; ++a) sel.position[a] = ops[i].picks[a];
      int by = -1;
      o.position = port_suggest(P, &sel, &by);
      o.by = by;
    } else {
      port_record(P, ops[i].af, ops[i].value);
      o.by = ops[i].af;
    }
    for (int a = 0; a < 3; ++a) {
      o.active[a] = P.active[a];
      o.duplicates[a] = P.duplicates[a];
      o.above[a] = P.above[a];
      o.below[a] = P.below[a];
      o.dos[a] = P.dos[a];
    }
  }
}

void launch_portfolio_trace(const PortDev& P, const PortOp* d_ops, int n, PortState* d_out, cudaStream_t s) {
  count_launch();
  k_portfolio_trace<<<1, 32, 0, s>>>(P, d_ops, n, d_out);
}

// The selection result from the merged partials (one thread): the
// first-candidate rule, the cross-shard merge pieces, then the resident
// loop's advance.
template <uint32_t MASK>
__device__ void select_publish(const SelCtx& c, const SelPart& f, double best, double lambda, double mean_var,
                               int cv_fallback, int gp_status, SelectDev* out, LoopDev* loop) {
  const int64_t ff = f.first;
  const long long fc = f.cnt;
  out->first_nan_mask = 0;
  for (int af = 0; af < 3; ++af) {
    out->best_nonnan_pos[af] = -1;
    out->best_nonnan_score[af] = 0.0;
  }
  for (int af = 0; af < 3; ++af) {
    int64_t pos = -1;
    double sc = 0.0;
    if ((c.af_mask & (1u << af)) && fc > 0) {
      // first-candidate rule (portfolio.hpp:52)
      bool first_nan = false;
      double s_first = 0.0;
      if (!f.finite || f.b[af].p == INT64_MAX) {
        s_first = score_of(af, c.mu[ff], sd_at(c, ff), best, lambda);
        first_nan = s_first != s_first;
      }
      if (first_nan || f.b[af].p == INT64_MAX) {
        pos = ff;
        sc = s_first;
      } else {
        pos = f.b[af].p;
        sc = f.b[af].s;
      }
      // the pieces a cross-shard merge needs to apply the same rule
      out->best_nonnan_pos[af] = f.b[af].p == INT64_MAX ? -1 : f.b[af].p;
      out->best_nonnan_score[af] = f.b[af].s;
      if (first_nan) out->first_nan_mask |= 1u << af;
    }
    out->position[af] = pos;
    out->score[af] = sc;
  }
  out->first_eligible = fc > 0 ? ff : -1;
  out->lambda = lambda;
  out->mean_variance = mean_var;
  out->best_std = best;
  out->n_candidates = (int64_t)fc;
  out->cv_fallback = cv_fallback;
  out->gp_status = gp_status;
  if (c.b.gthr) c.b.gthr[0] = c.b.gthr[1] = c.b.gthr[2] = 0ull;  // next selection starts afresh
  *c.b.counter = 0;
#ifdef GTC_SEL_TRACE
  g_sel_trace[2042][2] = gtc_globaltimer();
#endif
  if (loop && loop->nranks == 0) loop_advance(loop, out);  // (sharded: k_shard_merge advances)
#ifdef GTC_SEL_TRACE
  g_sel_trace[2042][3] = gtc_globaltimer();
#endif
}

// ---- the resident loop's bordered append, fused into the selection's last block
//
// Dynamic shared memory of a loop-mode selection (loop_append_smem): l, c, e,
// y, the substitution result and the pivot reciprocals [n_max] each, the
// pick's coordinates [kMaxDim], the virtual-lane partials [4][256] and the
// reduction scratch [32].
__host__ __device__ __forceinline__ size_t loop_append_doubles(int n_max) {
  return 6 * (size_t)n_max + kMaxDim + 4 * 256 + 32;
}

__device__ __forceinline__ double matern_rt(int nu, double r, double l, double s2) {
  return nu == 0 ? matern<0>(r, l, s2) : nu == 1 ? matern<1>(r, l, s2) : matern<2>(r, l, s2);
}

// cta_stats_beta over shared copies of y, c, e (n entries, the sum of y given):
// the same operations in the same order, so the same bits.
__device__ void stats_beta_staged(const GpDev& g, int n, double ysum, double y0, const double* ys, const double* cs,
                                  const double* es, double (*lanes)[256], double* red) {
  const double mean = n > 0 ? __ddiv_rn(ysum, (double)n) : 0.0;
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    double part = 0.0;
    for (int i = v; i < n; i += 256) {
      const double dv = __dadd_rn(ys[i], -mean);
      part = __dadd_rn(part, __dmul_rn(dv, dv));
    }
    lanes[0][v] = part;
  }
  double out[1];
  vsum256<1>(lanes, out, red);
  double stdv = 1.0;
  if (n > 1) {
    const double var = __ddiv_rn(out[0], (double)n);
    stdv = var > 0.0 ? sqrt(var) : 1.0;
  }
  if (threadIdx.x == 0) {
    g.sc->y_mean = mean;
    g.sc->y_std = stdv;
    g.sc->n = n;
  }
  const double shift = __dadd_rn(mean, -y0);
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    g.beta[i] = __ddiv_rn(__dadd_rn(cs[i], -__dmul_rn(shift, es[i])), stdv);
}

// Observation n0 = the step's valid pick, appended to the factor by the
// selection's last block right after loop_advance (no separate kernel, no
// launch boundary in the resident loop).  Every input is loaded at once (the
// pick's V column and coordinates, c, e, y, the scalars); then
//  - the V-column row (column_border_row: l = V(:, x*), the same fused
//    virtual-lane sums, the same 2^-8 pivot margin), or below the margin
//  - the exact bordered row (gp.hpp:105-121): Gram row with direct
//    differences, forward substitution as a column sweep -- each row's
//    subtractions in ascending column order, then times 1/L_ii, the operation
//    order of cta_forward_solve -- and |l|^2, l.c, l.e as virtual-lane sums
//    (== block_sum in the 256-thread GP kernels), so both rows are
//    bit-identical to k_gp_append's;
//  - then the standardisation and beta (cta_stats_beta's order).
// A failed exact pivot (x <= 0) sets status 1: the pass skips, the next
// selection halts the loop (kLoopPivot) and the host refactorises.
// `L` is the last block's shared copy of the loop state (already advanced).
// `col` (null: the exact row directly) is the pick's V column, rows
// `col_stride` apart; `xsrc` its coordinates, `x_stride` apart.
__device__ void loop_append(const LoopDev& L, double* dsm, const double* col, int64_t col_stride, const double* xsrc,
                            int64_t x_stride) {
  const GpDev& g = L.g;
  const int n0 = L.n0, d = L.sp.d, nm = g.n_max;
  double* ls = dsm;
  double* cs = ls + nm;
  double* es = cs + nm;
  double* ys = es + nm;
  double* xsol = ys + nm;
  double* rv = xsol + nm;
  double* xn = rv + nm;
  double (*lanes)[256] = reinterpret_cast<double (*)[256]>(xn + kMaxDim);
  double* red = xn + kMaxDim + 4 * 256;
  __shared__ double s_y0, s_jit;
  TRACE_AT(2040, 0);
  for (int q = threadIdx.x; q < n0; q += blockDim.x) {
    ls[q] = col ? __ldcg(col + (int64_t)q * col_stride) : 0.0;
    cs[q] = __ldcg(g.c + q);
    es[q] = __ldcg(g.e + q);
    ys[q] = __ldcg(g.y + q);
  }
  for (int t = threadIdx.x; t < d; t += blockDim.x) xn[t] = __ldcg(xsrc + (int64_t)t * x_stride);
  if (threadIdx.x == 0) {
    s_y0 = n0 == 0 ? L.y : __ldcg(&g.sc->y0);
    s_jit = __ldcg(&g.sc->jitter);
    ys[n0] = L.y;
  }
  __syncthreads();
  TRACE_AT(2040, 1);
  // append_prologue's effects: training row, its squared norm, the value, status
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int t = 0; t < d; ++t) {
      g.train_x[(int64_t)n0 * d + t] = xn[t];
      s = __dadd_rn(s, __dmul_rn(xn[t], xn[t]));
    }
    g.train_n2[n0] = s;
    g.y[n0] = L.y;
    g.sc->status = 0;
    g.sc->fail_row = -1;
    if (n0 == 0) g.sc->y0 = L.y;
  }
  // |l|^2, l.c, l.e and the sum of y[0, n0] in one virtual-lane reduction
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    double sq = 0.0, pc = 0.0, pe = 0.0, py = 0.0;
    for (int q = v; q < n0; q += 256) {
      const double l = ls[q];
      sq = __dadd_rn(sq, __dmul_rn(l, l));
      pc = __dadd_rn(pc, __dmul_rn(l, cs[q]));
      pe = __dadd_rn(pe, __dmul_rn(l, es[q]));
      py = __dadd_rn(py, ys[q]);
    }
    if (v == n0 % 256) py = __dadd_rn(py, ys[n0]);  // the new observation, last in its lane
    lanes[0][v] = sq;
    lanes[1][v] = pc;
    lanes[2][v] = pe;
    lanes[3][v] = py;
  }
  double r[4];
  vsum256<4>(lanes, r, red);
  const double diag = __dadd_rn(L.kp.s2, __dadd_rn(L.noise, s_jit));
  const double yr = __dadd_rn(L.y, -s_y0);
  double* Lrow = g.L + packed(n0);
  const double x = __dadd_rn(diag, -r[0]);
  const double* lrow = ls;
  if (!col || !(x > 0x1p-8 * diag)) {
    // ---- exact bordered row
    const double* xr = xn;
    for (int q = threadIdx.x; q < n0; q += blockDim.x) {
      const double* xa = g.train_x + (int64_t)q * d;
      double ss = 0.0;
      for (int t = 0; t < d; ++t) {
        const double dv = __dadd_rn(xa[t], -xr[t]);
        ss = __dadd_rn(ss, __dmul_rn(dv, dv));
      }
      ls[q] = matern_rt(L.kp.nu, sqrt(ss), L.kp.lengthscale, L.kp.s2);
      rv[q] = __drcp_rn(__ldg(g.L + packed(q) + q));
    }
    __syncthreads();
    // rows are owned by fixed threads, so each thread walks its rows of the
    // packed factor sequentially (L1 lines reused across iterations)
    for (int i = 0; i < n0; ++i) {
      const double xi = __dmul_rn(ls[i], rv[i]);
      if (threadIdx.x == 0) xsol[i] = xi;
      for (int q = threadIdx.x; q < n0; q += blockDim.x)
        if (q > i) ls[q] = __dadd_rn(ls[q], -__dmul_rn(__ldg(g.L + packed(q) + i), xi));
      __syncthreads();
    }
    for (int v = threadIdx.x; v < 256; v += blockDim.x) {
      double sq = 0.0;
      for (int q = v; q < n0; q += 256) sq = __dadd_rn(sq, __dmul_rn(xsol[q], xsol[q]));
      lanes[0][v] = sq;
    }
    double t1[1];
    vsum256<1>(lanes, t1, red);
    const double xe = __dadd_rn(diag, -t1[0]);
    if (xe <= 0.0) {  // Eigen LLT fails exactly when x <= 0 (a NaN pivot proceeds)
      if (threadIdx.x == 0) {
        g.sc->status = 1;
        g.sc->fail_row = n0;
      }
      __syncthreads();
      return;
    }
    const double lnn = sqrt(xe);
    for (int q = threadIdx.x; q < n0; q += blockDim.x) Lrow[q] = xsol[q];
    for (int v = threadIdx.x; v < 256; v += blockDim.x) {
      double pc = 0.0, pe = 0.0;
      for (int q = v; q < n0; q += 256) {
        pc = __dadd_rn(pc, __dmul_rn(xsol[q], cs[q]));
        pe = __dadd_rn(pe, __dmul_rn(xsol[q], es[q]));
      }
      lanes[0][v] = pc;
      lanes[1][v] = pe;
    }
    double t2[2];
    vsum256<2>(lanes, t2, red);
    if (threadIdx.x == 0) {
      Lrow[n0] = lnn;
      cs[n0] = __ddiv_rn(__dadd_rn(yr, -t2[0]), lnn);
      es[n0] = __ddiv_rn(__dadd_rn(1.0, -t2[1]), lnn);
      g.c[n0] = cs[n0];
      g.e[n0] = es[n0];
      if (col) ++g.sc->exact_rows;  // (a column attempt fell below the margin)
    }
  } else {
    const double lnn = sqrt(x);
    for (int q = threadIdx.x; q < n0; q += blockDim.x) Lrow[q] = lrow[q];
    if (threadIdx.x == 0) {
      Lrow[n0] = lnn;
      cs[n0] = __ddiv_rn(__dadd_rn(yr, -r[1]), lnn);
      es[n0] = __ddiv_rn(__dadd_rn(1.0, -r[2]), lnn);
      g.c[n0] = cs[n0];
      g.e[n0] = es[n0];
    }
  }
  __syncthreads();
  TRACE_AT(2040, 2);
  stats_beta_staged(g, n0 + 1, r[3], s_y0, ys, cs, es, lanes, red);
}

// Candidate-axis sharding: the shard's selection record for the all-gather
// (ShardHdr + the winners' coordinates and V columns, gtc_internal.h), from
// the local result select_publish just wrote.  Block-wide.
__device__ void shard_publish(const SelCtx& c, const LoopDev* L) {
  const SelectDev* s = c.out;
  ShardHdr* h = reinterpret_cast<ShardHdr*>(L->send);
  const int d = L->sp.d, n_max = L->g.n_max;
  const uint32_t mask = L->sel_mask;
  const int slots = shard_slots(mask);
  double* xs = reinterpret_cast<double*>(h + 1);
  double* xfirst = xs + slots * d;
  double* cols = xfirst + d;
  const int64_t off = L->offset;
  const bool live = s->n_candidates > 0;
  if (threadIdx.x == 0) {
    for (int af = 0; af < 3; ++af) {
      h->pos[af] = live && s->best_nonnan_pos[af] >= 0 ? s->best_nonnan_pos[af] + off : -1;
      h->score[af] = s->best_nonnan_score[af];
    }
    h->first = live && s->first_eligible >= 0 ? s->first_eligible + off : -1;
    h->count = s->n_candidates;
    h->nan_mask = live ? s->first_nan_mask : 0u;
    h->cv_fallback = s->cv_fallback;
    h->lambda = s->lambda;
    h->mean_var = s->mean_variance;
    h->best_std = s->best_std;
  }
  const int rows = L->n < n_max ? L->n : n_max;  // V rows [0, n) of the model
  int slot = 0;
  for (int af = 0; af < 3; ++af) {
    if (!(mask & (1u << af))) continue;
    const int64_t j = live ? s->best_nonnan_pos[af] : -1;
    if (j >= 0) {
      for (int t = threadIdx.x; t < d; t += blockDim.x) xs[slot * d + t] = L->sp.coords[(int64_t)t * L->sp.n_pad + j];
      const double* col = L->V + (j / kTile) * L->tile_stride + j % kTile;
      for (int q = threadIdx.x; q < rows; q += blockDim.x) cols[(int64_t)slot * n_max + q] = __ldcg(col + (int64_t)q * kTile);
    }
    ++slot;
  }
  const int64_t f = live ? s->first_eligible : -1;
  if (f >= 0)
    for (int t = threadIdx.x; t < d; t += blockDim.x) xfirst[t] = L->sp.coords[(int64_t)t * L->sp.n_pad + f];
}

template <uint32_t MASK>
__device__ void select_finish(const SelCtx& c, Best* b, int64_t first, int first_finite, long long cnt,
                              double best, double lambda, double mean_var, int cv_fallback, int gp_status) {
  __shared__ SelPart red[32];
  __shared__ bool is_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  SelPart v{{b[0], b[1], b[2]}, first, first_finite, cnt};
  v = sel_warp_reduce<MASK>(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    const SelPart none{{{0.0, INT64_MAX}, {0.0, INT64_MAX}, {0.0, INT64_MAX}}, INT64_MAX, 1, 0};
    v = sel_warp_reduce<MASK>(lane < nw ? red[lane] : none);
    if (lane == 0) {
      for (int af = 0; af < 3; ++af) {
        c.b.pscore[blockIdx.x * 3 + af] = v.b[af].s;
        c.b.ppos[blockIdx.x * 3 + af] = v.b[af].p;
      }
      c.b.pfirst[blockIdx.x] = v.first;
      c.b.pfinite[blockIdx.x] = v.finite;
      c.b.pcnt[blockIdx.x] = v.cnt;
      __threadfence();
      is_last = atomicAdd(c.b.counter, 1u) == gridDim.x - 1;
    }
    if (c.pf_table) {  // resident loop: warm L2 for the last block's lookups (any winner may be the pick)
#pragma unroll
      for (int af = 0; af < 3; ++af) {
        const int64_t p = v.b[af].p;
        if (!(MASK & (1u << af)) || p == INT64_MAX) continue;
        if (lane == 0) prefetch_l2(c.pf_table + p);
        const double* col = c.pf_V + (p / kTile) * c.pf_tile_stride + p % kTile;
        for (int q = lane; q < c.pf_rows; q += 32) prefetch_l2(col + (int64_t)q * kTile);
      }
    }
  }
  __syncthreads();
  SEL_MARK(5);
  if (!is_last) return;
  TRACE_AT(2042, 0);
  // last block: merge the per-block records (all loads in flight at once).
  // The result record and the loop state are built in shared memory (one
  // thread advances the loop: dependent global round trips would serialise)
  // and copied out block-wide.
  __shared__ SelectDev s_out;
  __shared__ LoopDev s_loop;
  static_assert(sizeof(LoopDev) % 8 == 0 && sizeof(SelectDev) % 8 == 0, "word copies");
  constexpr int kLoopWords = sizeof(LoopDev) / 8, kOutWords = sizeof(SelectDev) / 8;
  __threadfence();
  if (c.pf_c) {  // the fused append's inputs: into L2 while the merge runs (16 doubles per line)
    const int lines = (c.pf_rows + 16) / 16;
    for (int i = threadIdx.x; i < 3 * lines; i += blockDim.x)
      prefetch_l2((i < lines ? c.pf_c : i < 2 * lines ? c.pf_e : c.pf_y) + 16 * (i % lines));
  }
  if (c.loop)
    for (int i = threadIdx.x; i < kLoopWords; i += blockDim.x)
      reinterpret_cast<unsigned long long*>(&s_loop)[i] = __ldcg(reinterpret_cast<const unsigned long long*>(c.loop) + i);
  const SelPart none{{{0.0, INT64_MAX}, {0.0, INT64_MAX}, {0.0, INT64_MAX}}, INT64_MAX, 1, 0};
  SelPart f = none;
  for (int blk = threadIdx.x; blk < (int)gridDim.x; blk += blockDim.x) {
    SelPart y;
#pragma unroll
    for (int af = 0; af < 3; ++af)
      y.b[af] = Best{__ldcg(c.b.pscore + blk * 3 + af),
                     (int64_t)__ldcg(reinterpret_cast<const long long*>(c.b.ppos) + blk * 3 + af)};
    y.first = (int64_t)__ldcg(reinterpret_cast<const long long*>(c.b.pfirst) + blk);
    y.finite = __ldcg(c.b.pfinite + blk);
    y.cnt = __ldcg(c.b.pcnt + blk);
    f = sel_merge<MASK>(f, y);
  }
  f = sel_warp_reduce<MASK>(f);
  TRACE_AT(2042, 1);
  __syncthreads();  // red[] reuse
  if (lane == 0) red[warp] = f;
  __syncthreads();
  if (warp == 0) {
    f = sel_warp_reduce<MASK>(lane < nw ? red[lane] : none);
    if (lane == 0) select_publish<MASK>(c, f, best, lambda, mean_var, cv_fallback, gp_status, &s_out,
                                        c.loop ? &s_loop : nullptr);
  }
  __syncthreads();  // the result (thread 0) done
  for (int i = threadIdx.x; i < kOutWords; i += blockDim.x)
    reinterpret_cast<unsigned long long*>(c.out)[i] = reinterpret_cast<const unsigned long long*>(&s_out)[i];
  if (c.loop)
    for (int i = threadIdx.x; i < kLoopWords; i += blockDim.x)
      reinterpret_cast<unsigned long long*>(c.loop)[i] = reinterpret_cast<const unsigned long long*>(&s_loop)[i];
  if (c.host_sel) {  // direct read-back (gtc_observe): record + scalars, system fence, then the sequence word
    static_assert(sizeof(GpScalars) % 8 == 0, "word copies");
    for (int i = threadIdx.x; i < kOutWords; i += blockDim.x)
      reinterpret_cast<unsigned long long*>(c.host_sel)[i] = reinterpret_cast<const unsigned long long*>(&s_out)[i];
    for (int i = threadIdx.x; i < (int)(sizeof(GpScalars) / 8); i += blockDim.x)
      reinterpret_cast<unsigned long long*>(c.host_sc)[i] =
          __ldcg(reinterpret_cast<const unsigned long long*>(c.sc_src) + i);
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      *reinterpret_cast<volatile uint32_t*>(c.host_seq) = c.seq;
    }
  }
  if (c.loop && s_loop.nranks > 0) {
    __syncthreads();  // c.out / c.loop written
    shard_publish(c, c.loop);
  } else if (c.loop && s_loop.fused_append && s_loop.halt == kLoopRunning && s_loop.valid) {
    extern __shared__ double dsm[];
    const int64_t pos = s_loop.pos;
    loop_append(s_loop, dsm, s_loop.V + (pos / kTile) * s_loop.tile_stride + pos % kTile, kTile,
                s_loop.sp.coords + pos, s_loop.sp.n_pad);
  }
}


// Candidate-axis sharding: after the all-gather of the shard records, every
// shard merges them identically (best_candidate over the union,
// portfolio.hpp:32-61: the lowest eligible position is the first candidate and
// wins unconditionally when its score is NaN; else the highest non-NaN score,
// lowest position on ties), advances the replicated loop state (the visited
// mark lands on the owning shard only) and, for a valid pick, appends the
// bordered row from the winner's V column carried in its owner's record --
// the same column, coordinates and arithmetic as on one device, so the
// factor stays bit-identical on every shard.  The first-candidate case (NaN
// scores, no column shipped) leaves the exact row to the append kernel.
__global__ void __launch_bounds__(kCtaThreads) k_shard_merge(LoopDev* L) {
  __shared__ const double* s_x;
  __shared__ const double* s_col;
  pdl_begin();
  if (L->halt != kLoopRunning) return;
  const int d = L->sp.d, n_max = L->g.n_max;
  const uint32_t mask = L->sel_mask;
  const int slots = shard_slots(mask);
  const int64_t rb = L->rec_bytes;
  auto hdr = [&](int i) { return reinterpret_cast<const ShardHdr*>(L->recv + (int64_t)i * rb); };
  auto xs_of = [&](int i) { return reinterpret_cast<const double*>(hdr(i) + 1); };
  if (threadIdx.x == 0) {
    s_x = nullptr;
    s_col = nullptr;
    SelectDev* out = L->gsel;
    long long cnt = 0;
    int owner = -1;
    int64_t gfirst = INT64_MAX;
    for (int i = 0; i < L->nranks; ++i) {
      const ShardHdr* h = hdr(i);
      cnt += h->count;
      if (h->count > 0 && h->first >= 0 && h->first < gfirst) {
        gfirst = h->first;
        owner = i;
      }
    }
    int src[3] = {-1, -1, -1};  // shard whose record holds the winner's column (-1: first-candidate case)
    for (int af = 0; af < 3; ++af) {
      out->position[af] = -1;
      out->score[af] = 0.0;
      if (!(mask & (1u << af)) || owner < 0) continue;
      if (hdr(owner)->nan_mask & (1u << af)) {
        out->position[af] = gfirst;
        out->score[af] = CUDART_NAN;
        continue;
      }
      double bs = 0.0;
      int64_t bp = -1;
      for (int i = 0; i < L->nranks; ++i) {
        const ShardHdr* h = hdr(i);
        const int64_t p = h->pos[af];
        if (p < 0) continue;
        if (bp < 0 || h->score[af] > bs || (h->score[af] == bs && p < bp)) {
          bs = h->score[af];
          bp = p;
          src[af] = i;
        }
      }
      if (bp < 0) {  // every score NaN: the first candidate stands
        out->position[af] = gfirst;
        out->score[af] = CUDART_NAN;
      } else {
        out->position[af] = bp;
        out->score[af] = bs;
      }
    }
    const ShardHdr* h0 = hdr(0);
    out->lambda = h0->lambda;
    out->mean_variance = h0->mean_var;
    out->best_std = h0->best_std;
    out->n_candidates = cnt;
    out->cv_fallback = h0->cv_fallback;
    out->gp_status = 0;
    loop_advance(L, out);
    if (L->halt == kLoopRunning && L->valid) {
      const int by = L->rec[L->step - 1].by;
      int slot = 0;
      for (int af = 0; af < by; ++af) slot += (mask >> af) & 1u;
      const int o = src[by];
      if (o >= 0 && hdr(o)->pos[by] == L->pos) {
        s_x = xs_of(o) + slot * d;
        s_col = xs_of(o) + (slots + 1) * d + (int64_t)slot * n_max;
      } else {  // the first eligible candidate (owner's record)
        s_x = xs_of(owner) + slots * d;
      }
    }
  }
  __syncthreads();
  if (L->halt != kLoopRunning || !L->valid) return;
  for (int t = threadIdx.x; t < d; t += blockDim.x) L->xrec[(int64_t)(L->step - 1) * d + t] = s_x[t];
  // the bordered row from the winner's V column carried in its owner's record
  // (or, for the first-candidate case and below the margin, the exact row):
  // the same arithmetic as one device's fused append
  extern __shared__ double dsm[];
  loop_append(*L, dsm, s_col, 1, s_x, 1);
}

template <class K>
static void opt_in_smem(K kernel, size_t bytes);

void launch_shard_merge(LoopDev* loop, int nu, int n_max, cudaStream_t s) {
  (void)nu;
  count_launch();
  const size_t smem = loop_append_smem(n_max);
  opt_in_smem(k_shard_merge, smem);
  launch_pdl(k_shard_merge, dim3(1), dim3(kCtaThreads), smem, s, loop);
}

// ---------------------------------------------------- pruned selection
//
// Most of the selection's time is the FP64 erfc/exp/sqrt/div of every
// candidate's score, yet only the block's top few can be the argmax.  Phase 1
// computes a cheap FP32 UPPER BOUND ("key") of every candidate's FP64 score
// from the normal-tail (Mills ratio) inequalities, x >= 0:
//   2/(sqrt(x^2+4)+x) <= R(x) = (1-Phi(x))/phi(x) <= 4/(3x+sqrt(x^2+8))
// (Birnbaum 1942; Sampford 1953).  With h(z) = z Phi(z) + phi(z), EI = sd h(z):
//   z >= 0: h(z) = z + h(-z) <= z + phi(z) 4/(sqrt(z^2+4)+z)^2
//   z <  0: h(-x) = phi(x)(1 - x R(x)) <= phi(x) 4/(sqrt(x^2+4)+x)^2      (log2 key)
// PI = Phi(z):
//   z <  0: Phi(-x) = phi(x) R(x) <= phi(x) 4/(3x + sqrt(x^2+8))          (log2 key)
//   z >= 0: 1 - Phi(z) >= phi(z) 2/(sqrt(z^2+4)+z) =: q                 (key q, U = 1 - q)
// -LCB = lambda sd - mu with an FP32 sd rounded up                         (linear key)
// Tails are bounded in the log2 domain, so candidates far out in the tail
// (z << -13, where FP32 exp underflows) still prune against each other.
// Every key carries margins well above its FP32 evaluation error (<= 1e-3 in
// log2 up to |z| = 40, where the FP64 scores underflow to exactly 0) and above
// the rounding of the FP64 scores themselves (2^-30 relative, a 2^-1039 floor
// for subnormal results), and is rounded up.  The block then scores EXACTLY
// (the reference's FP64 formulas) its candidate with the largest key -> T,
// a score the block's best must reach, and scores exactly only candidates
// whose key does not prove score < T.  The block's best (max score, lowest
// position, NaN skipped) always passes, so the result is identical to scoring
// every candidate.  Non-finite inputs get +inf keys (always scored exactly).
constexpr int kSelPer = 8;  // candidates per thread per chunk (keys kept in registers)
constexpr float kLog2Slack = 0x1p-6f;  // log2-domain margin (1.1 % relative)
constexpr float kLog2Floor = -1039.0f;  // below this, subnormal rounding dominates
constexpr float kHalfLog2e = 0.72134752f;  // 1 / (2 ln 2)

// MUFU approximations (PTX: relative error <= 2^-22 for rcp/rsqrt/ex2,
// absolute <= 2^-22 for lg2 near 1, 2 ulp otherwise); all arguments here
// are normal floats and the margins above cover these errors.
__device__ __forceinline__ float f_rcp(float x) { float r; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float f_rsqrt(float x) { float r; asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float f_lg2(float x) { float r; asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float f_ex2(float x) { float r; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float f_sqrt(float x) { return x * f_rsqrt(x); }  // x > 0

// `spread` is the variance (run path, sd = sqrt(var) as strategies.hpp:385)
// or the std itself (best_candidate spans).  key[af] as described above;
// *pi_hi marks a PI key holding q (z >= 0).
// `base_ok`: |best -/+ lambda| < 1e30 (per block).  Inputs outside the
// guarded ranges (sd == 0, NaN, inf, |values| >= 1e30) get +inf keys.
template <uint32_t MASK, bool SD>
__device__ __forceinline__ void bound_keys(float* key, bool* pi_hi, double mu, double spread, bool base_ok,
                                           double bm_ei, double bp_pi, double lambda) {
  const float kInf = __int_as_float(0x7f800000);
  *pi_hi = false;
  const float sp = __double2float_rn(spread);
  const float mf = __double2float_rn(mu);  // NaN/inf/huge mu fail the guard
  if (!(base_ok && sp > (SD ? 1e-15f : 1e-30f) && sp < (SD ? 1e15f : 1e30f) && fabsf(mf) < 1e30f)) {
#pragma unroll
    for (int af = 0; af < 3; ++af) key[af] = kInf;  // exact scoring
    return;
  }
  const float rs = SD ? f_rcp(sp) : f_rsqrt(sp);  // 1 / sd
  const float sdf = SD ? sp : sp * rs;            // sd, relative error <= 2^-21
  if (MASK & 1u) {
    const double m = __dadd_rn(bm_ei, -mu);  // the reference's margin, exactly
    const float z = __double2float_rn(m) * rs;
    if (z >= 0.0f) {
      float t = 1e-38f;  // z > 13: >= phi(13) 4/(sqrt(173)+13)^2 = 4.7e-40
      if (z <= 13.0f) {
        const float den = f_sqrt(fmaf(z, z, 4.0f)) + z;
        t = 1.5957691f * f_ex2(-z * z * kHalfLog2e) * f_rcp(den * den);
      }
      const double u = fma((double)(sdf * t), 1.0 + 0x1p-8, m);
      key[0] = f_lg2(__double2float_ru(__dmul_rn(u, 1.0 + 0x1p-30))) + kLog2Slack;
    } else {
      const float x = -z, x2 = x * x;
      const float den = f_sqrt(x2 + 4.0f) + x;
      const float k = fmaf(-x2, kHalfLog2e, f_lg2(sdf * 1.5957691f * f_rcp(den * den))) + kLog2Slack;
      key[0] = x > 40.0f ? -kInf : fmaxf(k, kLog2Floor);  // x > 40: the FP64 score is exactly 0
    }
  }
  if (MASK & 2u) {
    const double m = __dadd_rn(bp_pi, -mu);
    const float z = __double2float_rn(m) * rs;
    if (z >= 0.0f) {  // q = lower bound of 1 - Phi(z); ex2 flushes to 0 beyond z ~ 13.2
      const float q = 0.79788456f * f_ex2(-z * z * kHalfLog2e) * f_rcp(f_sqrt(fmaf(z, z, 4.0f)) + z);
      key[1] = q * (1.0f - 0x1p-8f);  // decoded as 1 - q + 2^-50
      *pi_hi = true;
    } else {
      const float x = -z, x2 = x * x;
      const float k = fmaf(-x2, kHalfLog2e, f_lg2(1.5957691f * f_rcp(fmaf(3.0f, x, f_sqrt(x2 + 8.0f))))) + kLog2Slack;
      key[1] = x > 40.0f ? -kInf : fmaxf(k, kLog2Floor);  // x > 40: erfc underflows, score exactly 0
    }
  }
  if (MASK & 4u) {
    const double ls = __dmul_rn(lambda, __dmul_rn((double)sdf, 1.0 + 0x1p-20));
    const double slack = fma(__dadd_rn(fabs(mu), ls), 0x1p-40, 0x1p-1000);
    key[2] = __double2float_ru(__dadd_rn(__dadd_rn(ls, -mu), slack));
  }
}

// Ordering of keys for picking the block's threshold candidate.
__device__ __forceinline__ float key_rank(int af, float k, bool pi_hi) {
  return (af == 1 && pi_hi) ? 2.0f - k : k;
}

// Per-AF threshold in the form the survivor test uses.
struct Thr {
  double t;  // exact score reached in this block (-inf: none)
  float lt;  // float_rd(log2 t) for the log2-domain keys (-inf when t <= 0)
};

__device__ __forceinline__ bool may_reach(int af, float k, bool pi_hi, const Thr& th) {
  if (af == 2) return !((double)k < th.t);
  if (af == 1 && pi_hi) return !(__dadd_rn(__dadd_rn(1.0, -(double)k), 0x1p-50) < th.t);
  return !(k < th.lt);
}

template <uint32_t MASK, bool SD>
__device__ void select_pruned(const SelCtx& c, double best, double lambda, double mean_var, int cv_fallback,
                              int gp_status, int per) {
  __shared__ Best redb[32];
  __shared__ double s_thr[3];
  Best b[3] = {{0.0, INT64_MAX}, {0.0, INT64_MAX}, {0.0, INT64_MAX}};
  int64_t first = INT64_MAX;
  int first_finite = 1;
  long long cnt = 0;
  const double bm_ei = __dadd_rn(best, -lambda), bp_pi = __dadd_rn(best, lambda);
  const bool base_ok = fabs(bm_ei) < 1e30 && fabs(bp_pi) < 1e30;
  const double* spread = SD ? c.sdv : c.var;
  double thr[3] = {-CUDART_INF, -CUDART_INF, -CUDART_INF};  // running block threshold (exact scores)
  const int64_t chunk = (int64_t)per * blockDim.x;
  for (int64_t base = blockIdx.x * chunk; base < c.n; base += (int64_t)gridDim.x * chunk) {
    float key[kSelPer][3];
    uint32_t elig = 0, hi = 0;
    float top_r[3] = {-__int_as_float(0x7f800000), -__int_as_float(0x7f800000), -__int_as_float(0x7f800000)};
    int top_k[3] = {-1, -1, -1};
#pragma unroll
    for (int g = 0; g < kSelPer; g += 4) {  // four candidates' loads in flight
      double mu4[4], sp4[4];
      bool e4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t j = base + (int64_t)(g + q) * blockDim.x + threadIdx.x;
        const bool live = g + q < per && j < c.n;
        mu4[q] = live ? c.mu[j] : 0.0;
        sp4[q] = live ? spread[j] : 0.0;
        e4[q] = live && eligible(c, j);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = g + q;
        if (!e4[q]) continue;
        const int64_t j = base + (int64_t)k * blockDim.x + threadIdx.x;
        elig |= 1u << k;
        ++cnt;
        bool ph;
        bound_keys<MASK, SD>(key[k], &ph, mu4[q], sp4[q], base_ok, bm_ei, bp_pi, lambda);
        hi |= (uint32_t)ph << k;
        if (j < first) {  // (a thread meets its candidates in ascending position order)
          first = j;
          first_finite = 1;
#pragma unroll
          for (int af = 0; af < 3; ++af)
            if ((MASK & (1u << af)) && !(key[k][af] < __int_as_float(0x7f800000))) first_finite = 0;
        }
#pragma unroll
        for (int af = 0; af < 3; ++af) {
          if (!(MASK & (1u << af))) continue;
          const float r = key_rank(af, key[k][af], ph);
          if (key[k][af] < __int_as_float(0x7f800000) && (top_k[af] < 0 || r > top_r[af])) {  // finite inputs only
            top_r[af] = r;
            top_k[af] = k;
          }
        }
      }
    }
    // the candidate with the largest key, scored exactly, sets the threshold
#pragma unroll
    for (int af = 0; af < 3; ++af) {
      if (!(MASK & (1u << af))) continue;
      const Best t = block_best(top_k[af] < 0 ? Best{0.0, INT64_MAX}
                                              : Best{(double)top_r[af], base + (int64_t)top_k[af] * blockDim.x + threadIdx.x},
                                redb);
      if (threadIdx.x == 0) {
        double s = -CUDART_INF;
        if (t.p != INT64_MAX) {
          s = score_of(af, c.mu[t.p], sd_at(c, t.p), best, lambda);
          if (s != s) s = -CUDART_INF;
        }
        s_thr[af] = fmax(thr[af], s);
      }
    }
    __syncthreads();
    // survivors (keys that do not prove score < T), then exact scores for them
#pragma unroll
    for (int af = 0; af < 3; ++af) {
      if (!(MASK & (1u << af))) continue;
      thr[af] = s_thr[af];
      const Thr th{thr[af], thr[af] > 0.0 ? __double2float_rd(log2(thr[af])) : -__int_as_float(0x7f800000)};
      uint32_t surv = 0;
#pragma unroll
      for (int k = 0; k < kSelPer; ++k)
        if (((elig >> k) & 1u) && may_reach(af, key[k][af], (hi >> k) & 1u, th)) surv |= 1u << k;
#pragma unroll 1
      while (surv) {
        const int k = __ffs(surv) - 1;
        surv &= surv - 1;
        const int64_t j = base + (int64_t)k * blockDim.x + threadIdx.x;
        const double s = score_of(af, c.mu[j], sd_at(c, j), best, lambda);
        if (s == s) b[af] = better(b[af], Best{s, j});
      }
    }
    __syncthreads();  // s_thr reuse
  }
  select_finish<MASK>(c, b, first, first_finite, cnt, best, lambda, mean_var, cv_fallback, gp_status);
}

// Resident blocks per SM of the selection kernels: a single AF fits 64
// registers (two blocks), several AFs keep their keys in 128 (one block).
__host__ __device__ constexpr int sel_blocks_per_sm(uint32_t mask) { return (mask & (mask - 1)) ? 1 : 2; }

// lambda (strategies.hpp:404-418, acquisition.hpp:73-83) and best_std
// (gp.hpp:145) from the variance total: identical in every block.
struct SelSetup {
  double best, lambda, mean_var;
  int fallback;
};

__device__ __forceinline__ SelSetup sel_setup_vals(double s, long long cnt, const SelectParams& p, double y_mean,
                                                   double y_std) {
  SelSetup u;
  u.mean_var = cnt > 0 ? __ddiv_rn(s, (double)cnt) : 0.0;
  u.lambda = p.lambda_constant;
  u.fallback = 0;
  if (p.lambda_mode == 1) {
    if (!(p.f_best_raw > 0.0) || !(p.cv_mu_s > 0.0) || !(p.cv_var_s > 0.0)) {
      u.fallback = 1;
    } else {
      const double l = __ddiv_rn(__ddiv_rn(__dmul_rn(u.mean_var, p.f_best_raw), p.cv_mu_s), p.cv_var_s);
      u.lambda = l > 0.0 ? l : 0.0;
    }
  }
  u.best = __ddiv_rn(__dadd_rn(p.f_best_raw, -y_mean), y_std);
  return u;
}

__device__ __forceinline__ SelSetup sel_setup(const GpScalars* sc, const SelectParams& p, const VarSource& vs) {
  double s;
  long long cnt;
  var_source_read(vs, &s, &cnt);
  return sel_setup_vals(s, cnt, p, sc->y_mean, sc->y_std);
}

// Monotone map of non-NaN doubles to u64 (atomicMax of exact scores); 0 = none.
__device__ __forceinline__ unsigned long long ord_key(double d) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
  if (k == 0ull) return -CUDART_INF;
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

__device__ __forceinline__ Thr make_thr(double t) {
  return Thr{t, t > 0.0 ? __double2float_rd(log2(t)) : -__int_as_float(0x7f800000)};
}

// Upper bound keys of every score in a tile from its TileStats: EI and -LCB
// grow with the variance and fall with the mean, so (min mean, max variance)
// bounds them; PI = Phi((best + lambda - mu)/sd) is bounded with the minimum
// variance when best + lambda - min mean >= 0, else with the maximum.
template <uint32_t MASK>
__device__ __forceinline__ void tile_keys(const TileStats& ts, float* key, bool* pi_hi, bool base_ok, double bm_ei,
                                          double bp_pi, double lambda) {
  *pi_hi = false;
  if (!(ts.var_max >= 0.0)) {  // no candidates in the tile
#pragma unroll
    for (int af = 0; af < 3; ++af) key[af] = -__int_as_float(0x7f800000);
    return;
  }
  bool h;
  if (MASK & 5u) bound_keys<MASK & 5u, false>(key, &h, ts.mu_min, ts.var_max, base_ok, bm_ei, bp_pi, lambda);
  if (MASK & 2u) {
    float k2[3];
    const bool pos = __dadd_rn(bp_pi, -ts.mu_min) >= 0.0;
    bound_keys<2u, false>(k2, pi_hi, ts.mu_min, pos ? ts.var_min : ts.var_max, base_ok, bm_ei, bp_pi, lambda);
    key[1] = k2[1];
  }
}

// Selection for a resident run, one kernel:
//  - lambda and best_std from the run's fixed-point variance total (left by the
//    predictive pass or k_var_partials; VarAccum): every block computes the
//    same values without a grid barrier;
//  - tiles are dealt round-robin to blocks (candidates near the optimum
//    cluster in space, so contiguous ranges would make a few blocks do all
//    the exact scoring);
//  - each block bounds its tiles from their TileStats and scores exactly the
//    minimum-mean candidate of its best-keyed tile (recorded by the pass, so
//    no candidate loads): a threshold T that the block's best must reach;
//  - it keeps only tiles whose key reaches T, bounds their candidates and
//    scores exactly those whose key reaches T: the same argmax as scoring
//    every candidate (see select_pruned).
// The candidate count and the first eligible position come from the host's
// visited bookkeeping.
constexpr int kTileList = 512;  // tiles examined per block per round

template <uint32_t MASK>
__device__ __forceinline__ void select_run_body(const SelCtx& c, const GpScalars* sc, const SelectParams& p,
                                                const VarSource& vs, const TileStats* tstat, int ntiles,
                                                const SelSetup* pre = nullptr) {
  __shared__ int s_list[kTileList];
  __shared__ int s_n;
  SEL_MARK(0);
  const int G = gridDim.x;
  const int mine = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / G + 1 : 0;  // tiles of this block
  // this thread's first tile summary, loaded before the variance total (independent)
  TileStats ts0{};
  if ((int)threadIdx.x < mine) ts0 = tstat[blockIdx.x + G * threadIdx.x];
  // (its seed's eligibility too: the visited word load overlaps the setup below)
  const bool seed_ok0 = (int)threadIdx.x < mine && ts0.pos_seed >= 0 && eligible(c, ts0.pos_seed);
  // the first eligible candidate's inputs, loaded now by the block that owns it
  // (used at the end; keeps the load off the block's tail)
  const int64_t fp = p.first_eligible;
  const bool own_first = threadIdx.x == 0 && fp >= 0 && (int)((fp / kTile) % G) == (int)blockIdx.x;
  double f_mu = 0.0, f_var = 0.0;
  if (own_first) {
    f_mu = c.mu[fp];
    f_var = c.var[fp];
  }
#ifdef GTC_SEL_TRACE
  if (threadIdx.x == 0) { g_sel_trace[blockIdx.x][4] = gtc_globaltimer() + (unsigned long long)(ts0.mu_min == 12345.0); }
#endif
  // one thread per block reads the variance total and the GP scalars (every
  // block reads the same few words: one request per block, not per warp,
  // keeps the L2 slice that holds them from serialising ~5k requests)
  __shared__ SelSetup s_u;
  if (!pre) {
    if (threadIdx.x == 0) s_u = sel_setup(sc, p, vs);
    __syncthreads();
  }
  const SelSetup u = pre ? *pre : s_u;
  const double bm_ei = __dadd_rn(u.best, -u.lambda), bp_pi = __dadd_rn(u.best, u.lambda);
  const bool base_ok = fabs(bm_ei) < 1e30 && fabs(bp_pi) < 1e30;
  const float kInf = __int_as_float(0x7f800000);
  SEL_MARK(1);
  // ---- block threshold: the best exact score among the seeds of this block's
  // tiles (each tile's unvisited minimum-mean candidate, recorded by the pass
  // with its mean and variance, so no candidate loads); any exact score of an
  // eligible candidate is a valid threshold
  double sb[3] = {-CUDART_INF, -CUDART_INF, -CUDART_INF};
  for (int k = threadIdx.x; k < mine; k += blockDim.x) {
    const bool first_k = k == (int)threadIdx.x;
    const TileStats ts = first_k ? ts0 : tstat[blockIdx.x + G * k];
    if (ts.pos_seed < 0 || !(first_k ? seed_ok0 : eligible(c, ts.pos_seed))) continue;  // (marked after the pass)
    const double sd = sqrt(ts.var_seed);
#pragma unroll
    for (int af = 0; af < 3; ++af) {
      if (!(MASK & (1u << af))) continue;
      const double t = score_of(af, ts.mu_seed, sd, u.best, u.lambda);
      if (t == t) sb[af] = fmax(sb[af], t);
    }
  }
  __shared__ double s_sb[32][3];
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int af = 0; af < 3; ++af) {
      if (!(MASK & (1u << af))) continue;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sb[af] = fmax(sb[af], __shfl_xor_sync(0xffffffffu, sb[af], o));
      if (lane == 0) s_sb[warp][af] = sb[af];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int af = 0; af < 3; ++af) {
        if (!(MASK & (1u << af))) continue;
        double v = lane < nw ? s_sb[lane][af] : -CUDART_INF;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        sb[af] = v;
      }
    }
  }
  Thr th[3];
#pragma unroll
  for (int af = 0; af < 3; ++af) th[af] = Thr{sb[af], -kInf};  // (thread 0's values are the block's)
  // share thresholds across blocks: any block's exact score of an eligible
  // candidate is a valid threshold for every block (blocks far from the
  // optimum would otherwise score most of their candidates exactly)
  __shared__ double s_thr[3];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int af = 0; af < 3; ++af) {
      if (!(MASK & (1u << af))) continue;
      const unsigned long long prev =
          th[af].t > -CUDART_INF ? atomicMax(c.b.gthr + af, ord_key(th[af].t)) : __ldcg(c.b.gthr + af);
      s_thr[af] = fmax(th[af].t, ord_val(prev));
    }
  }
  __syncthreads();
#pragma unroll
  for (int af = 0; af < 3; ++af)
    if (MASK & (1u << af)) th[af] = make_thr(s_thr[af]);
  SEL_MARK(2);
  // ---- surviving tiles, their candidates, exact scores
  Best b[3] = {{0.0, INT64_MAX}, {0.0, INT64_MAX}, {0.0, INT64_MAX}};
  for (int g0 = 0; g0 < mine; g0 += kTileList) {
    const int g1 = min(mine, g0 + kTileList);
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int k = g0 + threadIdx.x; k < g1; k += blockDim.x) {
      const int t = blockIdx.x + G * k;
      const TileStats ts = k == (int)threadIdx.x ? ts0 : tstat[t];
      float key[3];
      bool hi;
      tile_keys<MASK>(ts, key, &hi, base_ok, bm_ei, bp_pi, u.lambda);
      bool keep = false;
#pragma unroll
      for (int af = 0; af < 3; ++af)
        if (MASK & (1u << af)) keep |= may_reach(af, key[af], hi, th[af]);
      if (keep) s_list[atomicAdd(&s_n, 1)] = t;
    }
    if (threadIdx.x < 3 && (MASK & (1u << threadIdx.x)))  // thresholds published since
      s_thr[threadIdx.x] = fmax(s_thr[threadIdx.x], ord_val(__ldcg(c.b.gthr + threadIdx.x)));
    __syncthreads();
#pragma unroll
    for (int af = 0; af < 3; ++af)
      if (MASK & (1u << af)) th[af] = make_thr(s_thr[af]);
    const int nl = s_n;
    for (int idx = threadIdx.x; idx < nl * kTile; idx += blockDim.x) {
      const int64_t j = (int64_t)s_list[idx / kTile] * kTile + idx % kTile;
      if (j >= c.n || !eligible(c, j)) continue;
      const double mu = c.mu[j], var = c.var[j];
      float key[3];
      bool hi;
      bound_keys<MASK, false>(key, &hi, mu, var, base_ok, bm_ei, bp_pi, u.lambda);
#pragma unroll
      for (int af = 0; af < 3; ++af) {
        if (!(MASK & (1u << af)) || !may_reach(af, key[af], hi, th[af])) continue;
        const double s = score_of(af, mu, sqrt(var), u.best, u.lambda);
        if (s == s) b[af] = better(b[af], Best{s, j});
      }
    }
    __syncthreads();  // s_list / s_n reuse
  }
  SEL_MARK(3);
  // the host-computed first eligible candidate lives in exactly one block
  int64_t first = INT64_MAX;
  int finite = 1;
  if (own_first) {
    float key[3];
    bool hi;
    bound_keys<MASK, false>(key, &hi, f_mu, f_var, base_ok, bm_ei, bp_pi, u.lambda);
    first = fp;
#pragma unroll
    for (int af = 0; af < 3; ++af)
      if ((MASK & (1u << af)) && !(key[af] < kInf)) finite = 0;
  }
  const long long cnt = (blockIdx.x == 0 && threadIdx.x == 0) ? (long long)p.n_candidates : 0;
  select_finish<MASK>(c, b, first, finite, cnt, u.best, u.lambda, u.mean_var, u.fallback, sc->status);
}

template <uint32_t MASK>
__global__ void __launch_bounds__(kSelectThreads, sel_blocks_per_sm(MASK))
    k_select(SelCtx c, const GpScalars* sc, SelectParams p, VarSource vs, const TileStats* tstat, int ntiles) {
  pdl_begin();
  SEL_MARK(7);
#ifdef GTC_SEL_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) g_sel_trace[2043][1] = g_sel_trace[2043][0];
#endif
  // Resident loop: the per-step inputs come from the loop state.  One thread
  // per block issues every load at once -- loop fields, GP scalars and BOTH
  // variance-accumulator generations (the generation is itself a loaded
  // value) -- so the block waits one L2 round trip, not a dependent chain;
  // it computes lambda / best_std and shares them through shared memory.
  __shared__ SelectParams s_p;
  __shared__ SelSetup s_pre;
  __shared__ int s_go, s_have;
  if (p.loop) {
    if (threadIdx.x == 0) {
      const LoopDev* lp = p.loop;
      const int halt = lp->halt, status = sc->status, nranks = lp->nranks, gen = lp->gen;
      const double f_best = lp->f_best, lconst = lp->lambda_constant, cvm = lp->cv_mu_s, cvv = lp->cv_var_s;
      const int64_t first = lp->first, count = lp->count;
      const int lmode = lp->lambda_mode;
      const double y_mean = sc->y_mean, y_std = sc->y_std;
      const VarAccum* gacc = lp->gacc;
      unsigned long long l[2][5];
#pragma unroll
      for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int k = 0; k < 5; ++k) l[g][k] = __ldcg(reinterpret_cast<const unsigned long long*>(vs.acc + g) + k);
      int go = halt == kLoopRunning;
      if (go && status != 0) {  // the last bordered row failed: the host refactorises
        if (blockIdx.x == 0) p.loop->halt = kLoopPivot;
        go = 0;
      }
      p.f_best_raw = f_best;
      p.first_eligible = first;
      p.n_candidates = count;
      p.lambda_mode = lmode;
      p.lambda_constant = lconst;
      p.cv_mu_s = cvm;
      p.cv_var_s = cvv;
      s_p = p;
      s_have = nranks == 0;
      if (go && nranks == 0) {
        unsigned long long lg[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) lg[k] = (gen & 1) ? l[1][k] : l[0][k];  // (no dynamic register indexing)
        s_pre = sel_setup_vals(limbs_value(lg, vs.s2), (long long)lg[4], p, y_mean, y_std);
      } else if (go) {  // sharded: the global total from every shard's gathered accumulators
        VarSource g = vs;
        g.gathered = gacc;
        g.n_gathered = nranks;
        g.gen = gen;
        double su;
        long long cn;
        var_source_read(g, &su, &cn);
        s_pre = sel_setup_vals(su, cn, p, y_mean, y_std);
        s_have = 1;
      }
      s_go = go;
    }
    __syncthreads();
    if (!s_go) return;
    p = s_p;
  }
  select_run_body<MASK>(c, sc, p, vs, tstat, ntiles, (p.loop && s_have) ? &s_pre : nullptr);
}


// Runs of a batch on the y axis (one AF mask per launch).
template <uint32_t MASK>
__global__ void __launch_bounds__(kSelectThreads, sel_blocks_per_sm(MASK))
    k_select_batch(const SelectRunArgs* __restrict__ args) {
  const SelectRunArgs& r = args[blockIdx.y];
  if (r.out == nullptr) return;
  const SelCtx c{r.mu, r.var, nullptr, r.visited, nullptr, r.p.excluded, r.p.n_excluded, r.n, r.p.af_mask, r.b, r.out};
  select_run_body<MASK>(c, r.sc, r.p, r.vs, r.tstat, (int)((r.n + kTile - 1) / kTile));
}

// (sum, count) of a variance source: a shard's local contribution to the
// global mean variance.
__global__ void k_var_totals(VarSource v, VarTotals* out) {
  double s;
  long long c;
  var_source_read(v, &s, &c);
  out->sum = s;
  out->count = c;
}

// Variance total over the unvisited candidates when the pass did not
// produce it for the current visited set (invalid observation, unmark).
__global__ void __launch_bounds__(kReduceThreads)
    k_var_partials(const double* __restrict__ var, const uint32_t* __restrict__ visited, int64_t n, double s2,
                   VarAccum* acc, VarAccum* acc_clear) {
  __shared__ double red[32];
  __shared__ long long redl[32];
  accum_clear(acc_clear);
  double s;
  long long c;
  var_partial(var, visited, n, red, redl, &s, &c);
  if (threadIdx.x == 0) accum_add(acc, s, c, s2);
}

template <uint32_t MASK>
__global__ void __launch_bounds__(kSelectThreads, sel_blocks_per_sm(MASK)) k_best_candidate(SelCtx c, double best, double lambda, int per) {
  select_pruned<MASK, true>(c, best, lambda, 0.0, 0, 0, per);
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

// Opt-in to large dynamic shared memory: the attribute is raised to the
// largest size requested so far per kernel and device (a driver call only
// when the requirement grows, not on every launch of the observe step).
template <class K>
static void opt_in_smem(K kernel, size_t bytes) {
  // the 48 KB default covers static + dynamic shared memory, so every kernel
  // with dynamic shared memory opts in once (the static arrays of the GP
  // kernels alone take 12-25 KB)
  if (bytes == 0) return;
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, size_t>> set_to;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  const std::pair<const void*, int> key{(const void*)kernel, dev};
  for (auto& e : set_to) {
    if (e.first != key) continue;
    if (e.second >= bytes) return;
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess)
      e.second = bytes;
    return;
  }
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess)
    set_to.push_back({key, bytes});
}

// 1: right-looking factor in shared memory when it fits (default); 0: the
// left-looking bordered rows (GTC_FACTOR=left, diagnostics).
static int g_factor_mode = [] {
  const char* e = std::getenv("GTC_FACTOR");
  return (e && std::string(e) == "left") ? 0 : 1;
}();
void set_factor_mode(int mode) { g_factor_mode = mode; }
int factor_mode() { return g_factor_mode; }

void launch_gp_factor(const GpDev& g, KernelParams k, double noise, double jitter, int n,
                      cudaStream_t s) {
  count_launch();
  const size_t rl = sizeof(double) * ((size_t)even_up(packed(n)) + 3 * (size_t)n);
  if (g_factor_mode == 1 && n > 0 && rl <= 200 * 1024) {  // right-looking, the factor in shared memory
    switch (k.nu) {
      case 0: opt_in_smem(k_gp_factor_rl<0>, rl); k_gp_factor_rl<0><<<1, kFactorThreads, rl, s>>>(g, k, noise, jitter, n); break;
      case 1: opt_in_smem(k_gp_factor_rl<1>, rl); k_gp_factor_rl<1><<<1, kFactorThreads, rl, s>>>(g, k, noise, jitter, n); break;
      default: opt_in_smem(k_gp_factor_rl<2>, rl); k_gp_factor_rl<2><<<1, kFactorThreads, rl, s>>>(g, k, noise, jitter, n); break;
    }
    return;
  }
  bool staged;
  const size_t sm = cta_smem_bytes(g.n_max, n, &staged);
  const int st = staged ? 1 : 0;
  switch (k.nu) {
    case 0: opt_in_smem(k_gp_factor<0>, sm); k_gp_factor<0><<<1, kCtaThreads, sm, s>>>(g, k, noise, jitter, n, st); break;
    case 1: opt_in_smem(k_gp_factor<1>, sm); k_gp_factor<1><<<1, kCtaThreads, sm, s>>>(g, k, noise, jitter, n, st); break;
    default: opt_in_smem(k_gp_factor<2>, sm); k_gp_factor<2><<<1, kCtaThreads, sm, s>>>(g, k, noise, jitter, n, st); break;
  }
}

AppendArgs make_append_args(const GpDev& g, KernelParams k, double noise, const SpaceDev& sp, int64_t pos,
                             const double* x_explicit, double y_new, int n0, uint32_t* visited_mark,
                             size_t* smem_bytes) {
  bool staged;
  *smem_bytes = cta_smem_bytes(g.n_max, n0 + 1, &staged);
  return AppendArgs{g, k, noise, sp, pos, x_explicit, y_new, n0, visited_mark, staged ? 1 : 0};
}

void launch_gp_append(const GpDev& g, KernelParams k, double noise, const SpaceDev& sp,
                      int64_t pos, const double* x_explicit, double y_new, int n0,
                      uint32_t* visited_mark, cudaStream_t s, const double* V, int64_t tile_stride) {
  count_launch();
  size_t sm;
  AppendArgs a = make_append_args(g, k, noise, sp, pos, x_explicit, y_new, n0, visited_mark, &sm);
  a.V = V;
  a.tile_stride = tile_stride;
  switch (k.nu) {
    case 0: opt_in_smem(k_gp_append<0>, sm); launch_pdl(k_gp_append<0>, 1, kCtaThreads, sm, s, a); break;
    case 1: opt_in_smem(k_gp_append<1>, sm); launch_pdl(k_gp_append<1>, 1, kCtaThreads, sm, s, a); break;
    default: opt_in_smem(k_gp_append<2>, sm); launch_pdl(k_gp_append<2>, 1, kCtaThreads, sm, s, a); break;
  }
}

void launch_gp_append_batch(const AppendArgs* d_args, int count, int nu, size_t smem, cudaStream_t s) {
  count_launch();
  switch (nu) {
    case 0: opt_in_smem(k_gp_append_batch<0>, smem); k_gp_append_batch<0><<<count, kCtaThreads, smem, s>>>(d_args); break;
    case 1: opt_in_smem(k_gp_append_batch<1>, smem); k_gp_append_batch<1><<<count, kCtaThreads, smem, s>>>(d_args); break;
    default: opt_in_smem(k_gp_append_batch<2>, smem); k_gp_append_batch<2><<<count, kCtaThreads, smem, s>>>(d_args); break;
  }
}



void launch_gp_truncate(const GpDev& g, int n, cudaStream_t s) {
  count_launch();
  k_gp_truncate<<<1, kCtaThreads, 0, s>>>(g, n);
}

static bool deep_pass(int64_t tiles) {
  static const int off = [] {
    const char* e = std::getenv("GTC_PASS_DEEP");
    return e && e[0] == '0';
  }();
  return !off && tiles < 4 * (int64_t)sm_count();
}

template <int R, int NU>
static void extend_impl(const ExtendArgs& a, int64_t tiles, cudaStream_t s) {
  const size_t sm = sizeof(double) * ((size_t)(R + 1) * (a.n0 + R) + (size_t)R * a.g.d + R + 8);
  if (R == 1 && deep_pass(tiles)) {
    opt_in_smem(k_extend_deep<NU>, sm);
    launch_pdl(k_extend_deep<NU>, dim3((unsigned)tiles), dim3(kExtendThreads), sm, s, a);
    return;
  }
  opt_in_smem(k_extend<R, NU>, sm);
  launch_pdl(k_extend<R, NU>, dim3((unsigned)tiles), dim3(kExtendThreads), sm, s, a);
}

// ------------------------------------------------------------ V rebuild on the FP64 tensor cores
//
// The full forward substitution V = L^-1 K* (gp.hpp:163-164) for every
// candidate -- the initial fit, refits after jitter escalation and the
// stand-alone predict -- as ONE pass that writes V once, instead of n/8
// streaming passes that re-read the growing prefix (k_extend<8>: ~n^2/16 rows
// of HBM traffic).  Blocked by 8-row panels exactly like k_extend<8>:
//   acc  = sum_{m < n0} L[n0+t][m] v_m       (ascending FMA chain)
//   num  = k(x_{n0+t}, x) - acc               (expansion-form kernel)
//   num -= L[n0+t][n0+s] * v_s, s < t         (multiply, then subtract)
//   v    = num / L[n0+t][n0+t]
// The panel contraction `acc` is the dense, GEMM-shaped part: FP64 mma.sync
// m8n8k4 (DMMA), A = 8 panel rows x 4 columns of L, B = 4 V rows x 8
// candidates, D = 8 x 8 accumulators.  A chain of DMMAs over k is
// bit-identical to the ascending FMA chain (tools/dmma_order.cu: 0 of 262,144
// elements differ), so this kernel writes exactly the V of the streaming
// rebuild.  One warp owns 8 candidates: its V block [n][8] stays in shared
// memory (B fragments: 4 rows x 64 B, conflict-free), its panel triangle runs
// in the D-fragment layout (row t on lanes 4t..4t+3, broadcast by shuffle),
// and warps never synchronise with each other.  L is read through L1 (the
// warps of a CTA walk the same panels).  The posterior (mean, variance, tile
// summaries, variance total) then comes from the R = 0 final pass, whose
// FMA order over the rows is the streaming rebuild's.
constexpr int kRbMaxWarps = 12;  // warps per CTA, shared-memory permitting
constexpr int kRbGroups = 2;     // column groups of 8 candidates per warp (DMMA chains sharing A)
constexpr int kRbCands = 8 * kRbGroups;

// Shared memory: two staged L panels [8][ld] (+ their training rows, norms
// and pivot reciprocals), then per warp its V blocks [kRbGroups][n][8], the
// candidate coordinates [d][kRbCands], their squared norms and a transpose
// scratch [kRbGroups][8][8].
__host__ __device__ __forceinline__ int rebuild_ld(int n) { return ((n + 8 + 15) / 16) * 16 + 4; }
__host__ __device__ __forceinline__ size_t rebuild_panel_doubles(int n, int d) {
  return (size_t)8 * rebuild_ld(n) + (size_t)8 * d + 8 + 8;
}
__host__ __device__ __forceinline__ size_t rebuild_warp_doubles(int n, int d) {
  return (size_t)kRbCands * n + (size_t)kRbCands * d + kRbCands + 64 * kRbGroups;
}

struct RebuildArgs {
  SpaceDev sp;
  GpDev g;
  double* V;
  int64_t tile_stride;
  int n;
  double lengthscale, s2;
};

__device__ __forceinline__ double coord1(const SpaceDev& sp, int t, int64_t j) {
  if (sp.cidx) return __ldg(sp.ctab + t * 256 + sp.cidx[(int64_t)t * sp.n_pad + j]);
  return __ldg(sp.coords + (int64_t)t * sp.n_pad + j);
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Panel n0 (rows n0 .. n0+7 of the packed factor, their training rows and
// squared norms) into a staging buffer, asynchronously (cp.async).
__device__ void rebuild_stage_panel(const GpDev& g, int n, int n0, double* buf) {
  const int ld = rebuild_ld(n), d = g.d;
  const int r = min(8, n - n0);
  for (int t = 0; t < r; ++t) {
    const double* src = g.L + packed(n0 + t);
    for (int q = threadIdx.x; q <= n0 + t; q += blockDim.x) cp_async8(buf + t * ld + q, src + q);
  }
  double* xr = buf + 8 * ld;
  for (int i = threadIdx.x; i < r * d; i += blockDim.x) cp_async8(xr + i, g.train_x + (int64_t)n0 * d + i);
  for (int t = threadIdx.x; t < r; t += blockDim.x) cp_async8(xr + 8 * d + t, g.train_n2 + n0 + t);
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int NU>
__global__ void __launch_bounds__(kRbMaxWarps * 32, 1) k_rebuild(RebuildArgs a) {
  constexpr int G = kRbGroups;
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int n = a.n, d = a.sp.d, ld = rebuild_ld(n);
  const size_t pd = rebuild_panel_doubles(n, d);
  double* Vs = sm + 2 * pd + (size_t)w * rebuild_warp_doubles(n, d);  // [G][n][8] this warp's V blocks
  double* cx = Vs + (size_t)kRbCands * n;                              // [d][kRbCands] coordinates
  double* cn2 = cx + (size_t)kRbCands * d;                             // [kRbCands] squared norms
  double* T = cn2 + kRbCands;                                          // [G][8][8] transpose scratch
  const int64_t c0 = ((int64_t)blockIdx.x * W + w) * kRbCands;         // first candidate of the warp
  const bool active = c0 < a.sp.n_pad;
  const double linv = __drcp_rn(a.lengthscale);
  rebuild_stage_panel(a.g, n, 0, sm);
  if (active) {
    for (int idx = lane; idx < kRbCands * d; idx += 32)
      cx[idx] = coord1(a.sp, idx / kRbCands, c0 + idx % kRbCands);
    __syncwarp();
    if (lane < kRbCands) {  // sequential in t (extend_body's c0n2)
      double s = 0.0;
      for (int t = 0; t < d; ++t) s = __dadd_rn(s, __dmul_rn(cx[t * kRbCands + lane], cx[t * kRbCands + lane]));
      cn2[lane] = s;
    }
    __syncwarp();
  }
  const int row = lane >> 2, kq = lane & 3;  // fragment coordinates: D rows `row`, cols 2kq, 2kq+1
  const int col = 2 * kq;
  const bool tri = lane < kRbCands;          // transposed layout: lane = candidate
  const int tg = lane >> 3, tc = lane & 7;   // its group and column
  double* Vg = a.V + (c0 / kTile) * a.tile_stride + c0 % kTile;  // row m at Vg + m * kTile
  int buf = 0;
  for (int n0 = 0; n0 < n; n0 += 8, buf ^= 1) {
    const int r = min(8, n - n0);
    const bool live = row < r;
    // the next panel streams in while this one is used
    if (n0 + 8 < n) rebuild_stage_panel(a.g, n, n0 + 8, sm + (buf ^ 1) * pd);
    if (n0 + 8 < n) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const double* Lp = sm + buf * pd;
    const double* Lr = Lp + row * ld;  // this thread's A row (rows past r: stale, masked)
    const double* xr = Lp + 8 * ld;    // [r][d] training rows, then [r] norms
    if (active) {
      // ---- kernel values of the panel rows in the fragment layout
      // (gp.hpp:176-179 expansion form, extend_body's order); independent of
      // the contraction below, so their latency overlaps it
      double kv[G][2];
#pragma unroll
      for (int g = 0; g < G; ++g) kv[g][0] = kv[g][1] = 0.0;
      if (live) {
        const double xn2 = xr[8 * d + row];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int cc = 8 * g + col;
          double dot0 = 0.0, dot1 = 0.0;
          for (int t = 0; t < d; ++t) {
            const double xv = xr[row * d + t];
            dot0 = __dadd_rn(dot0, __dmul_rn(xv, cx[t * kRbCands + cc]));
            dot1 = __dadd_rn(dot1, __dmul_rn(xv, cx[t * kRbCands + cc + 1]));
          }
          const double d20 = __dadd_rn(__dadd_rn(__dmul_rn(-2.0, dot0), xn2), cn2[cc]);
          const double d21 = __dadd_rn(__dadd_rn(__dmul_rn(-2.0, dot1), xn2), cn2[cc + 1]);
          kv[g][0] = matern_q<NU>(sqrt(fmax(d20, 0.0)), a.lengthscale, linv, a.s2);
          kv[g][1] = matern_q<NU>(sqrt(fmax(d21, 0.0)), a.lengthscale, linv, a.s2);
        }
      }
      // ---- panel contraction on the tensor cores: rows m < n0, G chains
      // sharing each A fragment (four k-steps of fragments loaded together)
      double acc[G][2];
#pragma unroll
      for (int g = 0; g < G; ++g) acc[g][0] = acc[g][1] = 0.0;
      const double* Ap = Lr + kq;
      const double* Bp = Vs + kq * 8 + row;  // group g's B fragment: + g * 8n, row m0 + kq at + m0 * 8
      int m0 = 0;
      for (; m0 + 16 <= n0; m0 += 16) {
        double av[4], bv[4][G];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          av[u] = live ? Ap[m0 + 4 * u] : 0.0;
#pragma unroll
          for (int g = 0; g < G; ++g) bv[u][g] = Bp[(size_t)g * 8 * n + (m0 + 4 * u) * 8];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int g = 0; g < G; ++g)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[g][0]), "+d"(acc[g][1])
                         : "d"(av[u]), "d"(bv[u][g]));
      }
      for (; m0 < n0; m0 += 4) {
        const double av = live ? Ap[m0] : 0.0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const double bv = Bp[(size_t)g * 8 * n + m0 * 8];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[g][0]), "+d"(acc[g][1])
                       : "d"(av), "d"(bv));
        }
      }
      // ---- num = k - acc, transposed through shared memory: lane c < 8G
      // takes candidate c's eight panel rows
#pragma unroll
      for (int g = 0; g < G; ++g)
        *reinterpret_cast<double2*>(T + g * 64 + row * 8 + col) =
            make_double2(__dadd_rn(kv[g][0], -acc[g][0]), __dadd_rn(kv[g][1], -acc[g][1]));
      __syncwarp();
      // ---- the panel triangle, one candidate per lane, in registers
      // (k_extend<8>'s order: subtract the earlier rows of the panel in
      // ascending order, then divide; quot_rn == __ddiv_rn)
      if (tri) {
        double num[8], v[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) num[t] = t < r ? T[tg * 64 + t * 8 + tc] : 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (t >= r) break;
          const double* Lt = Lp + t * ld + n0;
          double x = num[t];
#pragma unroll
          for (int s2 = 0; s2 < t; ++s2) x = __dadd_rn(x, -__dmul_rn(Lt[s2], v[s2]));
          v[t] = quot_rn(x, Lt[t], __drcp_rn(Lt[t]));
          Vs[(size_t)tg * 8 * n + (n0 + t) * 8 + tc] = v[t];
          Vg[(int64_t)(n0 + t) * kTile + lane] = v[t];
        }
      }
      __syncwarp();
    }
    __syncthreads();  // this buffer is free for the stage after next
  }
}

// 0: streaming rebuild (k_extend<8>, n/8 launches, prefix from HBM);
// 1: tensor-core rebuild (k_rebuild + one final pass).  GTC_REBUILD=stream
// selects 0 (diagnostics).  (A third variant -- one CTA per tile running all
// of its 8-row panels back to back so the prefix would come from L2 -- was
// measured and dropped: 36 % L2 hit rate, 10.7 GB of DRAM reads, 9.6 ms.)
// 2: k_kstar + the 32-row DFMA passes (k_extend_wide); 3: the same on FP64
// mma.sync (k_extend_wide_mma); 4 (default): the persistent 64-row DMMA
// passes (k_extend_pm; falls back to 2 when its rows of L do not fit).
static int g_rebuild_mode = [] {
  const char* e = std::getenv("GTC_REBUILD");
  if (e && std::string(e) == "stream") return 0;
  if (e && std::string(e) == "dmma") return 1;
  if (e && std::string(e) == "wide") return 2;
  if (e && std::string(e) == "widemma") return 3;
  if (e && std::string(e) == "pmma") return 4;
  return 4;
}();
void set_rebuild_mode(int mode) { g_rebuild_mode = mode; }

int rebuild_mode() { return g_rebuild_mode; }

// Wide streaming rebuild (k_extend_wide, 32 rows per pass), the final pass
// with the posterior.  false = not taken (mode off, or the staging does not
// fit shared memory for this n).
bool rebuild_wide_taken(const SpaceDev& sp, int n) {
  if ((g_rebuild_mode < 2 || g_rebuild_mode > 4) || n <= 0) return false;
  if (g_rebuild_mode == 3 && sizeof(double) * wm_smem_doubles(n) > 200 * 1024) return false;
  return sizeof(double) * wide_smem_doubles(n, sp.d) <= 200 * 1024;
}

// Every kernel value k(x_t, x), t < n, at full occupancy, into the V rows
// they become (needs only the training coordinates: the fit runs it beside
// the factorisation on a second stream).
void launch_kstar(const SpaceDev& sp, const GpDev& g, KernelParams k, double* V, int64_t tile_stride, int n,
                  cudaStream_t s) {
  const int64_t tiles = sp.n_pad / kTile;
  {
    count_launch();
    ExtendArgs a{sp, g, V, tile_stride, 0, 0, 0, 0, k.lengthscale, k.s2};
    const dim3 grid((unsigned)tiles, (unsigned)((n + kKstarRows - 1) / kKstarRows));
    const bool regs = sp.d <= 8;
    switch (k.nu) {
      case 0: regs ? k_kstar<0, 8><<<grid, kExtendThreads, 0, s>>>(a, n) : k_kstar<0, 0><<<grid, kExtendThreads, 0, s>>>(a, n); break;
      case 1: regs ? k_kstar<1, 8><<<grid, kExtendThreads, 0, s>>>(a, n) : k_kstar<1, 0><<<grid, kExtendThreads, 0, s>>>(a, n); break;
      default: regs ? k_kstar<2, 8><<<grid, kExtendThreads, 0, s>>>(a, n) : k_kstar<2, 0><<<grid, kExtendThreads, 0, s>>>(a, n); break;
    }
  }
}

bool launch_rebuild_wide(const SpaceDev& sp, const GpDev& g, KernelParams k, double* V, int64_t tile_stride, int n,
                         double* mu, double* var, const VarPartials* vp, TileStats* tstat, cudaStream_t s,
                         bool kstar_done) {
  if (!rebuild_wide_taken(sp, n)) return false;
  const bool mma = g_rebuild_mode == 3;
  // the 64-row passes when their rows of L fit shared memory (n <= ~380), else the 32-row passes
  const int pm_last = (n - 1) / kPmRows * kPmRows;
  const bool pm = g_rebuild_mode == 4 && sizeof(double) * pm_smem_doubles(pm_last, false) <= 224 * 1024;
  // (the B rings when every pass's staging fits with them: n <= ~250)
  const bool pm_ring = pm && kPmRingSteps > 0 && sizeof(double) * pm_smem_doubles(pm_last, true) <= 224 * 1024;
  const size_t need = sizeof(double) * wide_smem_doubles(n, sp.d);
  const int64_t tiles = sp.n_pad / kTile;
  if (!kstar_done) launch_kstar(sp, g, k, V, tile_stride, n, s);
  if (pm) {  // persistent 64-row DMMA passes (V rows only), then the posterior from an r = 0 pass
    static int sms = [] {
      int dev = 0, v = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
      return v > 0 ? v : 148;
    }();
    const int64_t groups = sp.n_pad / 16;
    // group counters of this rebuild's passes (the GP store's, so runs
    // rebuilding concurrently on their own streams do not share them)
    const int passes = (n + kPmRows - 1) / kPmRows;
    int* ctr = g.work;
    if (!ctr || passes > kGpWork) return false;
    cudaMemsetAsync(ctr, 0, passes * sizeof(int), s);
    for (int n0 = 0, pass = 0; n0 < n; n0 += kPmRows, ++pass) {
      count_launch();
      ExtendArgs a{sp, g, V, tile_stride, n0, std::min(kPmRows, n - n0), 0, 0, k.lengthscale, k.s2};
      const size_t smem = sizeof(double) * pm_smem_doubles(n0, pm_ring);
      opt_in_smem(k_extend_pm, smem);
      const unsigned grid = (unsigned)std::min<int64_t>(sms, (groups + kPmWarps - 1) / kPmWarps);
      k_extend_pm<<<grid, kPmWarps * 32, smem, s>>>(a, ctr + pass, pm_ring ? 1 : 0);
    }
    launch_extend(sp, g, k, V, tile_stride, n, 0, true, mu, var, false, vp, tstat, s);
    return true;
  }
  if (mma) {  // DMMA passes (V rows only), then the posterior from an r = 0 pass
    for (int n0 = 0; n0 < n; n0 += kWideRows) {
      count_launch();
      ExtendArgs a{sp, g, V, tile_stride, n0, std::min(kWideRows, n - n0), 0, 0, k.lengthscale, k.s2};
      const size_t smem = sizeof(double) * wm_smem_doubles(n0);
      opt_in_smem(k_extend_wide_mma, smem);
      const unsigned grid = (unsigned)(sp.n_pad / (8 * kWmWarps));
      k_extend_wide_mma<<<grid, kWmWarps * 32, smem, s>>>(a);
    }
    launch_extend(sp, g, k, V, tile_stride, n, 0, true, mu, var, false, vp, tstat, s);
    return true;
  }
  for (int n0 = 0; n0 < n; n0 += kWideRows) {
    count_launch();
    const int r = std::min(kWideRows, n - n0);
    const bool final = n0 + r == n;
    ExtendArgs a{sp, g, V, tile_stride, n0, r, final ? 1 : 0, 0, k.lengthscale, k.s2, mu, var,
                 vp ? vp->visited : nullptr, (vp && final) ? vp->acc : nullptr, vp ? vp->acc_clear : nullptr,
                 final ? tstat : nullptr};
    a.kstar = 1;
    const size_t smem = sizeof(double) * wide_smem_doubles(n0, sp.d, true);
    switch (k.nu) {
      case 0: opt_in_smem(k_extend_wide<0>, need); k_extend_wide<0><<<(unsigned)tiles, kExtendThreads, smem, s>>>(a); break;
      case 1: opt_in_smem(k_extend_wide<1>, need); k_extend_wide<1><<<(unsigned)tiles, kExtendThreads, smem, s>>>(a); break;
      default: opt_in_smem(k_extend_wide<2>, need); k_extend_wide<2><<<(unsigned)tiles, kExtendThreads, smem, s>>>(a); break;
    }
  }
  return true;
}

// V rows [0, n) of every candidate (no posterior).  Returns false when the
// tensor-core path is off or the per-warp block does not fit shared memory.
bool launch_rebuild(const SpaceDev& sp, const GpDev& g, KernelParams k, double* V, int64_t tile_stride, int n,
                    cudaStream_t s) {
  if (g_rebuild_mode != 1 || n <= 0) return false;
  constexpr size_t kBudget = 224 * 1024;
  const size_t fixed = sizeof(double) * 2 * rebuild_panel_doubles(n, sp.d);
  const size_t per_warp = sizeof(double) * rebuild_warp_doubles(n, sp.d);
  if (fixed + per_warp > kBudget) return false;
  const int64_t groups = sp.n_pad / kRbCands;  // (n_pad is a multiple of 256)
  const int W = (int)std::min<int64_t>({(int64_t)kRbMaxWarps, (int64_t)((kBudget - fixed) / per_warp), groups});
  const size_t smem = fixed + per_warp * W;
  count_launch();
  const RebuildArgs a{sp, g, V, tile_stride, n, k.lengthscale, k.s2};
  const unsigned grid = (unsigned)((groups + W - 1) / W);
  switch (k.nu) {
    case 0: opt_in_smem(k_rebuild<0>, smem); k_rebuild<0><<<grid, W * 32, smem, s>>>(a); break;
    case 1: opt_in_smem(k_rebuild<1>, smem); k_rebuild<1><<<grid, W * 32, smem, s>>>(a); break;
    default: opt_in_smem(k_rebuild<2>, smem); k_rebuild<2><<<grid, W * 32, smem, s>>>(a); break;
  }
  return true;
}

void launch_extend(const SpaceDev& sp, const GpDev& g, KernelParams k, double* V,
                   int64_t tile_stride, int n0, int r, bool final, double* mu, double* var,
                   bool check_status, const VarPartials* vp, TileStats* tstat, cudaStream_t s) {
  count_launch();
  ExtendArgs a{sp, g, V, tile_stride, n0, r, final ? 1 : 0, check_status ? 1 : 0,
               k.lengthscale, k.s2, mu, var, vp ? vp->visited : nullptr,
               (vp && final) ? vp->acc : nullptr, vp ? vp->acc_clear : nullptr, final ? tstat : nullptr};
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

template <int NU>
static void extend_loop_impl(const ExtendArgs& a, int64_t tiles, cudaStream_t s) {
  extend_impl<1, NU>(a, tiles, s);
}

void launch_extend_loop(const ExtendArgs& a, int64_t tiles, int nu, cudaStream_t s) {
  count_launch();
  switch (nu) {
    case 0: extend_loop_impl<0>(a, tiles, s); break;
    case 1: extend_loop_impl<1>(a, tiles, s); break;
    default: extend_loop_impl<2>(a, tiles, s); break;
  }
}

ExtendArgs make_pass_args(const SpaceDev& sp, const GpDev& g, KernelParams k, double* V, int64_t tile_stride,
                          int n0, double* mu, double* var, const VarPartials* vp, TileStats* tstat) {
  return ExtendArgs{sp, g, V, tile_stride, n0, 1, 1, 1, k.lengthscale, k.s2, mu, var, vp ? vp->visited : nullptr,
                    vp ? vp->acc : nullptr, vp ? vp->acc_clear : nullptr, tstat};
}

void launch_extend_batch(const ExtendArgs* d_args, int count, int64_t tiles, int nu, int max_n0, int d,
                         cudaStream_t s) {
  count_launch();
  const size_t sm = sizeof(double) * ((size_t)2 * (max_n0 + 1) + (size_t)d + 1 + 8);
  const dim3 grid((unsigned)tiles, (unsigned)count);
  switch (nu) {
    case 0: opt_in_smem(k_extend_batch<0>, sm); k_extend_batch<0><<<grid, kExtendThreads, sm, s>>>(d_args); break;
    case 1: opt_in_smem(k_extend_batch<1>, sm); k_extend_batch<1><<<grid, kExtendThreads, sm, s>>>(d_args); break;
    default: opt_in_smem(k_extend_batch<2>, sm); k_extend_batch<2><<<grid, kExtendThreads, sm, s>>>(d_args); break;
  }
}

// Copies scattered device records into one contiguous buffer (one read-back
// for a whole batch of runs).
__global__ void k_gather(const GatherDesc* __restrict__ d, unsigned char* __restrict__ dst) {
  const GatherDesc g = d[blockIdx.x];
  for (uint32_t i = threadIdx.x; i < g.bytes; i += blockDim.x) dst[g.dst_offset + i] = g.src[i];
}

void launch_gather(const GatherDesc* d_descs, int count, unsigned char* dst, cudaStream_t s) {
  count_launch();
  k_gather<<<count, 128, 0, s>>>(d_descs, dst);
}

void launch_mark_batch(const MarkDesc* d_marks, int count, cudaStream_t s) {
  count_launch();
  k_mark_batch<<<(count + 127) / 128, 128, 0, s>>>(d_marks, count);
}

void launch_prior(double* mu, double* var, int64_t n, double s2, TileStats* tstat, cudaStream_t s) {
  count_launch();
  k_prior<<<148, 256, 0, s>>>(mu, var, n, s2, tstat);
}

void launch_mark(uint32_t* visited, int64_t pos, int set, cudaStream_t s, VarAccum* acc, const double* var,
                 double s2) {
  count_launch();
  k_mark<<<1, 1, 0, s>>>(visited, pos, set, acc, var, s2);
}

void launch_varsum(const double* var, const uint32_t* visited, int64_t n, double* ps, int64_t* pc,
                   unsigned int* counter, VarTotals* totals, cudaStream_t s) {
  count_launch();
  k_varsum<<<reduce_blocks(n), kReduceThreads, 0, s>>>(var, visited, n, ps, pc, counter, totals);
}

void launch_var_totals(const VarSource& src, VarTotals* out, cudaStream_t s) {
  count_launch();
  k_var_totals<<<1, 1, 0, s>>>(src, out);
}

void launch_var_partials(const double* var, int64_t n, double s2, const VarPartials& vp, cudaStream_t s) {
  count_launch();
  k_var_partials<<<reduce_blocks(n), kReduceThreads, 0, s>>>(var, vp.visited, n, s2, vp.acc, vp.acc_clear);
}

// One wave of kSelectThreads-blocks, `per` candidates per thread per chunk.
static void select_geometry(int64_t n, uint32_t mask, int* per, int* grid) {
  const int64_t sms = (int64_t)sel_blocks_per_sm(mask) * sm_count();  // resident blocks
  *per = (int)std::max<int64_t>(1, std::min<int64_t>(kSelPer, (n + sms * kSelectThreads - 1) / (sms * kSelectThreads)));
  const int64_t chunk = (int64_t)*per * kSelectThreads;
  *grid = (int)std::max<int64_t>(1, std::min<int64_t>({(n + chunk - 1) / chunk, sms, (int64_t)kMaxReduceGrid}));
}

// Threads per selection block: a block handles ceil(tiles / grid) tiles, so
// when there are fewer tiles than resident 512-thread blocks (small spaces,
// one tile per block) most threads would idle; 128-thread blocks hold far
// fewer SM resources per tile (several concurrent runs share the device).
// The argmax does not depend on the block size (max with the lowest-position
// tie rule; thresholds are exact scores).
static int select_threads(int ntiles, uint32_t mask) {
  static const int forced = [] {
    const char* e = std::getenv("GTC_SELECT_THREADS");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 128 || forced == 256 || forced == 512) return forced;
  return ntiles < sel_blocks_per_sm(mask) * sm_count() ? 128 : kSelectThreads;
}

void launch_select(const double* mu, const double* var, const uint32_t* visited, int64_t n,
                   const GpScalars* sc, SelectParams p, const VarSource& vs, const TileStats* tstat,
                   const ReduceBufs& b, SelectDev* out, cudaStream_t s, int fused_append_n_max) {
  count_launch();
  SelCtx c{mu,     var,   nullptr,          visited,          nullptr, p.excluded, p.n_excluded, n,
           p.af_mask, b,   out,              p.loop,           p.pf_table, p.pf_V, p.pf_tile_stride, p.pf_rows,
           p.pf_gp[0], p.pf_gp[1], p.pf_gp[2], p.host_sel, p.host_sc, p.host_seq, p.seq, sc};
  const size_t smem = fused_append_n_max > 0 ? loop_append_smem(fused_append_n_max) : 0;
  const uint32_t mask = (p.af_mask & 7u) ? (p.af_mask & 7u) : 7u;
  const int ntiles = (int)((n + kTile - 1) / kTile);
  static const int grid_override = [] {
    const char* e = std::getenv("GTC_SELECT_GRID");  // diagnostics (tools/sel_bench.cu)
    return e ? std::atoi(e) : 0;
  }();
  const int want = grid_override > 0 ? grid_override : sel_blocks_per_sm(mask) * sm_count();
  const int grid = std::max(1, std::min({ntiles, want, kMaxReduceGrid}));
  const int threads = select_threads(ntiles, mask);
#define GTC_SELECT_CASE(M)                                                           \
  case M:                                                                                 \
    opt_in_smem(k_select<M>, smem);                                                         \
    launch_pdl(k_select<M>, dim3(grid), dim3(threads), smem, s, c, sc, p, vs, tstat, ntiles); \
    break;
  switch (mask) {  // launch errors surface through the caller's cudaGetLastError()
    GTC_SELECT_CASE(1)
    GTC_SELECT_CASE(2)
    GTC_SELECT_CASE(3)
    GTC_SELECT_CASE(4)
    GTC_SELECT_CASE(5)
    GTC_SELECT_CASE(6)
    default: GTC_SELECT_CASE(7)
  }
#undef GTC_SELECT_CASE
}

size_t loop_append_smem(int n_max) { return sizeof(double) * loop_append_doubles(n_max); }

void launch_select_batch(const SelectRunArgs* d_args, int count, uint32_t mask, int64_t n, cudaStream_t s) {
  count_launch();
  const uint32_t m = (mask & 7u) ? (mask & 7u) : 7u;
  const int ntiles = (int)((n + kTile - 1) / kTile);
  const int grid = std::max(1, std::min({ntiles, sel_blocks_per_sm(m) * sm_count(), kMaxReduceGrid}));
  const dim3 g((unsigned)grid, (unsigned)count);
  const int t = select_threads(ntiles, m);
  switch (m) {
    case 1: k_select_batch<1><<<g, t, 0, s>>>(d_args); break;
    case 2: k_select_batch<2><<<g, t, 0, s>>>(d_args); break;
    case 3: k_select_batch<3><<<g, t, 0, s>>>(d_args); break;
    case 4: k_select_batch<4><<<g, t, 0, s>>>(d_args); break;
    case 5: k_select_batch<5><<<g, t, 0, s>>>(d_args); break;
    case 6: k_select_batch<6><<<g, t, 0, s>>>(d_args); break;
    default: k_select_batch<7><<<g, t, 0, s>>>(d_args); break;
  }
}

void launch_best_candidate(const double* mu, const double* sd, const uint8_t* excluded, int64_t n,
                           int af, double best_std, double lambda, const ReduceBufs& b, SelectDev* out,
                           cudaStream_t s) {
  count_launch();
  SelCtx c{mu, nullptr, sd, nullptr, excluded, nullptr, 0, n, 1u << af, b, out};
  int per, grid;
  select_geometry(n, 1u << af, &per, &grid);
  if (af == 0) k_best_candidate<1><<<grid, kSelectThreads, 0, s>>>(c, best_std, lambda, per);
  else if (af == 1) k_best_candidate<2><<<grid, kSelectThreads, 0, s>>>(c, best_std, lambda, per);
  else k_best_candidate<4><<<grid, kSelectThreads, 0, s>>>(c, best_std, lambda, per);
}

void launch_scores(const double* mu, const double* sd, int64_t n, int af, double best_std,
                   double lambda, double* out, cudaStream_t s) {
  count_launch();
  k_scores<<<reduce_blocks(n), kReduceThreads, 0, s>>>(mu, sd, n, af, best_std, lambda, out);
}

}  // namespace gtc
