// sm_100a kernels of the device search-space enumeration.
//
// Reference: SearchSpace::enumerate_valid + EnumeratedSpace
// (/root/reference/proj/include/gridtune/search_space.hpp:120-166,216-245):
// walk the Cartesian grid in canonical order (mixed radix, first parameter
// most significant), keep the configurations that satisfy every restriction
// (restriction.hpp:416-504), and give each kept configuration the normalised
// coordinates rank / (k - 1).
//
// Here (1) k_enum_mask evaluates the compiled restriction programs (postfix,
// restriction.cpp) for every canonical index and writes a validity bitmask
// (one ballot per warp = one 32-bit word), counting the valid indices per
// block; (2) k_enum_scan turns the block counts into offsets; (3)
// k_enum_compact writes, in ascending canonical order, the valid indices and
// their coordinates (SoA, from host-computed exact rank/(k-1) tables) plus the
// 1-byte rank copy the predictive pass reads.  Bit-exactness: the programs use
// IEEE +,-,*,/ without contraction, fmod (exact), and IEEE comparisons (false
// against NaN), exactly the reference's double semantics; string comparisons
// were decided on the host.
#include <cuda_runtime.h>

#include <math_constants.h>

#include <algorithm>
#include <climits>
#include <cstdint>

#include "gtc_internal.h"
#include "restriction.hpp"

namespace gtc {

constexpr int kEnumThreads = 256;

__device__ __forceinline__ bool enum_valid(const EnumInstr* code, int n_code, const double* values,
                                           const int32_t* val_off, const uint8_t* str_tab, const int32_t* radix,
                                           const int* rank) {
  double st[kEnumMaxStack];
  int sp = 0;
  for (int pc = 0; pc < n_code; ++pc) {
    const EnumInstr ins = code[pc];
    switch (ins.op) {
      case kOpConst: st[sp++] = ins.k; break;
      case kOpParam: st[sp++] = values[val_off[ins.a] + rank[ins.a]]; break;
      case kOpStrTable: {
        const int ra = ins.a == 255 ? 0 : rank[ins.a];
        const int rb = ins.b == 255 ? 0 : rank[ins.b];
        const int kb = ins.b == 255 ? 1 : radix[ins.b];
        st[sp++] = __ldg(str_tab + ins.c + ra * kb + rb) ? 1.0 : 0.0;
        break;
      }
      case kOpNeg: st[sp - 1] = -st[sp - 1]; break;
      case kOpNot: st[sp - 1] = st[sp - 1] != 0.0 ? 0.0 : 1.0; break;
      case kOpEnd:
        if (st[--sp] == 0.0) return false;
        break;
      default: {
        const double b = st[--sp], a = st[sp - 1];
        double r;
        switch (ins.op) {
          case kOpAdd: r = __dadd_rn(a, b); break;
          case kOpSub: r = __dsub_rn(a, b); break;
          case kOpMul: r = __dmul_rn(a, b); break;
          case kOpDiv: r = __ddiv_rn(a, b); break;
          case kOpMod: r = fmod(a, b); break;
          case kOpEq: r = a == b; break;
          case kOpNe: r = a != b; break;
          case kOpLt: r = a < b; break;
          case kOpLe: r = a <= b; break;
          case kOpGt: r = a > b; break;
          case kOpGe: r = a >= b; break;
          case kOpAnd: r = (a != 0.0 && b != 0.0); break;
          default: r = (a != 0.0 || b != 0.0); break;  // kOpOr
        }
        st[sp - 1] = r;
      }
    }
  }
  return true;
}

// Mixed-radix decode of a canonical index (search_space.hpp:77-84).
__device__ __forceinline__ void enum_ranks(uint32_t idx, const int32_t* radix, int d, int* rank) {
  for (int i = d - 1; i >= 0; --i) {
    const uint32_t k = (uint32_t)radix[i];
    rank[i] = (int)(idx % k);
    idx /= k;
  }
}

// Block b owns the contiguous words [b * wpb_words, (b + 1) * wpb_words) in both
// passes, so block offsets follow canonical order.
__global__ void __launch_bounds__(kEnumThreads)
    k_enum_mask(EnumDev e, int64_t wpb_words, uint32_t* __restrict__ mask, int64_t* __restrict__ block_counts) {
  extern __shared__ __align__(16) unsigned char smem[];
  EnumInstr* code = reinterpret_cast<EnumInstr*>(smem);
  double* values = reinterpret_cast<double*>(code + e.n_code);
  int32_t* val_off = reinterpret_cast<int32_t*>(values + e.n_values);
  int32_t* radix = val_off + e.d;
  const EnumInstr* gcode = static_cast<const EnumInstr*>(e.code);
  for (int i = threadIdx.x; i < e.n_code; i += blockDim.x) code[i] = gcode[i];
  for (int i = threadIdx.x; i < e.n_values; i += blockDim.x) values[i] = e.values[i];
  for (int i = threadIdx.x; i < e.d; i += blockDim.x) {
    val_off[i] = e.val_off[i];
    radix[i] = e.radix[i];
  }
  __syncthreads();
  int rank[kEnumMaxParams];
  long long count = 0;
  const int64_t words = (e.total + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = blockIdx.x * wpb_words, w1 = min(words, w0 + wpb_words);
  for (int64_t w = w0 + (threadIdx.x >> 5); w < w1; w += blockDim.x / 32) {
    const int64_t idx = w * 32 + lane;
    bool ok = false;
    if (idx < e.total) {
      enum_ranks((uint32_t)idx, radix, e.d, rank);
      ok = enum_valid(code, e.n_code, values, val_off, e.str_tab, radix, rank);
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, ok);
    if (lane == 0) {
      mask[w] = bits;
      count += __popc(bits);
    }
  }
  // block total (lane 0 of each warp holds its count)
  __shared__ long long wsum[kEnumThreads / 32];
  if (lane == 0) wsum[threadIdx.x >> 5] = count;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = 0;
    for (int i = 0; i < kEnumThreads / 32; ++i) s += wsum[i];
    block_counts[blockIdx.x] = s;
  }
}

// Exclusive scan of the per-block counts (one block; fixed order) and the total.
__global__ void k_enum_scan(int64_t* counts, int nblocks, int64_t* total) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  // each thread scans a contiguous chunk
  const int per = (nblocks + blockDim.x - 1) / blockDim.x;
  const int lo = min(nblocks, t * per), hi = min(nblocks, lo + per);
  int64_t s = 0;
  for (int i = lo; i < hi; ++i) s += counts[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int64_t run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const int64_t v = part[i];
      part[i] = run;
      run += v;
    }
    *total = run;
  }
  __syncthreads();
  int64_t run = part[t];
  for (int i = lo; i < hi; ++i) {
    const int64_t v = counts[i];
    counts[i] = run;
    run += v;
  }
}

// Writes the valid canonical indices in ascending order with their
// coordinates: the block's words in rounds of one word per warp, each round's
// positions from the block offset + the popcounts of the preceding words.
__global__ void __launch_bounds__(kEnumThreads)
    k_enum_compact(EnumDev e, int64_t wpb_words, const uint32_t* __restrict__ mask,
                   const int64_t* __restrict__ block_offsets, int64_t n_pad, uint64_t* __restrict__ ids,
                   double* __restrict__ coords, uint8_t* __restrict__ cidx) {
  __shared__ int32_t radix[kEnumMaxParams], noff[kEnumMaxParams];
  __shared__ long long wsum[kEnumThreads / 32];
  __shared__ long long base;
  for (int i = threadIdx.x; i < e.d; i += blockDim.x) {
    radix[i] = e.radix[i];
    noff[i] = e.val_off[i];
  }
  if (threadIdx.x == 0) base = block_offsets[blockIdx.x];
  __syncthreads();
  const int64_t words = (e.total + 31) / 32;
  const int wpb = blockDim.x / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int rank[kEnumMaxParams];
  const int64_t w0 = blockIdx.x * wpb_words, w1 = min(words, w0 + wpb_words);
  for (int64_t r0 = w0; r0 < w1; r0 += wpb) {
    const int64_t w = r0 + wid;
    const uint32_t bits = w < w1 ? mask[w] : 0u;
    if (lane == 0) wsum[wid] = __popc(bits);
    __syncthreads();
    long long before = base;
    for (int i = 0; i < wid; ++i) before += wsum[i];
    long long round_total = 0;
    for (int i = 0; i < wpb; ++i) round_total += wsum[i];
    const bool mine = (bits >> lane) & 1u;
    if (mine) {
      const int64_t pos = before + __popc(bits & ((1u << lane) - 1u));
      const int64_t idx = w * 32 + lane;
      ids[pos] = (uint64_t)idx;
      enum_ranks((uint32_t)idx, radix, e.d, rank);
      for (int t = 0; t < e.d; ++t) {
        coords[(int64_t)t * n_pad + pos] = e.normtab[noff[t] + rank[t]];
        if (cidx) cidx[(int64_t)t * n_pad + pos] = (uint8_t)rank[t];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) base += round_total;
    __syncthreads();
  }
}

// Grid and words per block shared by both passes (contiguous word ranges).
// ---- initial-sample snap (sampling.hpp:98-117) ------------------------------
// For every design point, the position with the smallest squared distance
// d2 = sum_j (p_j - c_j)^2 (accumulated in j order, no contraction, exactly
// the reference's loop) and the lowest position on ties (its strict `<` scan).
constexpr int kSnapThreads = 256;
constexpr int kSnapGroup = 8;  // design points per pass (registers)

struct SnapBest {
  double d2;
  long long pos;
};
__device__ __forceinline__ SnapBest snap_min(SnapBest a, SnapBest b) {
  return (b.d2 < a.d2 || (b.d2 == a.d2 && b.pos < a.pos)) ? b : a;
}

__global__ void __launch_bounds__(kSnapThreads)
    k_snap_partial(SpaceDev sp, const double* __restrict__ pts, int n_pts, SnapBest* __restrict__ partial) {
  __shared__ SnapBest red[kSnapThreads / 32][kSnapGroup];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int g0 = 0; g0 < n_pts; g0 += kSnapGroup) {
    SnapBest best[kSnapGroup];
#pragma unroll
    for (int q = 0; q < kSnapGroup; ++q) best[q] = SnapBest{CUDART_INF, LLONG_MAX};
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < sp.n; j += (int64_t)gridDim.x * blockDim.x) {
      double d2[kSnapGroup];
#pragma unroll
      for (int q = 0; q < kSnapGroup; ++q) d2[q] = 0.0;
      for (int t = 0; t < sp.d; ++t) {
        const double c = sp.cidx ? __ldg(sp.ctab + t * 256 + sp.cidx[(int64_t)t * sp.n_pad + j])
                                 : sp.coords[(int64_t)t * sp.n_pad + j];
#pragma unroll
        for (int q = 0; q < kSnapGroup; ++q) {
          if (g0 + q < n_pts) {
            const double diff = __dsub_rn(pts[(g0 + q) * sp.d + t], c);
            d2[q] = __dadd_rn(d2[q], __dmul_rn(diff, diff));
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kSnapGroup; ++q) best[q] = snap_min(best[q], SnapBest{d2[q], (long long)j});
    }
#pragma unroll
    for (int q = 0; q < kSnapGroup; ++q) {
      for (int o = 16; o > 0; o >>= 1) {
        SnapBest other{__shfl_xor_sync(0xffffffffu, best[q].d2, o), __shfl_xor_sync(0xffffffffu, best[q].pos, o)};
        best[q] = snap_min(best[q], other);
      }
      if (lane == 0) red[wid][q] = best[q];
    }
    __syncthreads();
    if (threadIdx.x < kSnapGroup && g0 + (int)threadIdx.x < n_pts) {
      SnapBest b = red[0][threadIdx.x];
      for (int w = 1; w < kSnapThreads / 32; ++w) b = snap_min(b, red[w][threadIdx.x]);
      partial[(int64_t)blockIdx.x * n_pts + g0 + threadIdx.x] = b;
    }
    __syncthreads();
  }
}

__global__ void k_snap_merge(const SnapBest* __restrict__ partial, int blocks, int n_pts, int64_t* out) {
  const int q = blockIdx.x;  // one block per design point
  SnapBest b{CUDART_INF, LLONG_MAX};
  for (int i = threadIdx.x; i < blocks; i += blockDim.x) b = snap_min(b, partial[(int64_t)i * n_pts + q]);
  for (int o = 16; o > 0; o >>= 1) {
    SnapBest other{__shfl_xor_sync(0xffffffffu, b.d2, o), __shfl_xor_sync(0xffffffffu, b.pos, o)};
    b = snap_min(b, other);
  }
  __shared__ SnapBest red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    SnapBest m = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = snap_min(m, red[w]);
    out[q] = m.pos == LLONG_MAX ? 0 : (int64_t)m.pos;  // (the reference scan starts at position 0)
  }
}

int snap_partial_blocks(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + kSnapThreads - 1) / kSnapThreads, 148 * 4));
}

void launch_snap(const SpaceDev& sp, const double* pts, int n_pts, void* partial, int64_t* out, cudaStream_t s) {
  const int blocks = snap_partial_blocks(sp.n);
  k_snap_partial<<<blocks, kSnapThreads, 0, s>>>(sp, pts, n_pts, static_cast<SnapBest*>(partial));
  k_snap_merge<<<n_pts, 256, 0, s>>>(static_cast<const SnapBest*>(partial), blocks, n_pts, out);
}

static void enum_geometry(int64_t total, int* grid, int64_t* wpb_words) {
  const int64_t words = (total + 31) / 32;
  const int64_t wpb = kEnumThreads / 32;
  const int64_t g = std::max<int64_t>(1, std::min<int64_t>((words + wpb - 1) / wpb, 148 * 8));
  int64_t per = (words + g - 1) / g;
  per = (per + wpb - 1) / wpb * wpb;
  *wpb_words = per;
  *grid = (int)std::max<int64_t>(1, (words + per - 1) / per);
}

int64_t launch_enumerate_mask(const EnumDev& e, uint32_t* mask, int64_t* block_counts, int64_t* total_valid,
                              cudaStream_t s) {
  int grid;
  int64_t wpb_words;
  enum_geometry(e.total, &grid, &wpb_words);
  const size_t sm = sizeof(EnumInstr) * e.n_code + sizeof(double) * e.n_values + sizeof(int32_t) * 2 * e.d + 16;
  if (sm + 8 * 1024 > 48 * 1024)  // the 48 KB default covers static + dynamic shared memory
    cudaFuncSetAttribute(k_enum_mask, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_enum_mask<<<grid, kEnumThreads, sm, s>>>(e, wpb_words, mask, block_counts);
  k_enum_scan<<<1, 1024, 0, s>>>(block_counts, grid, total_valid);
  return grid;
}

void launch_enumerate_compact(const EnumDev& e, const uint32_t* mask, const int64_t* block_offsets, int64_t n_pad,
                              uint64_t* ids, double* coords, uint8_t* cidx, cudaStream_t s) {
  int grid;
  int64_t wpb_words;
  enum_geometry(e.total, &grid, &wpb_words);
  k_enum_compact<<<grid, kEnumThreads, 0, s>>>(e, wpb_words, mask, block_offsets, n_pad, ids, coords, cidx);
}

}  // namespace gtc
