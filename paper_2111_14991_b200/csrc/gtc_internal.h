// Internal declarations shared by the kernels (gtc_kernels.cu) and the C ABI
// host layer (gtc_capi.cu).  Not part of the public ABI (include/gridtune_cuda.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gtc {

// Candidates per tile.  V (= L^-1 K*, one row per GP observation) is stored
// tile-major: V[tile][row][kTile], so one tile's rows are one contiguous
// n_max*kTile*8-byte stream and an appended row is a contiguous 2 KB store
// per tile.  See DESIGN.md "Data layout in HBM".
constexpr int kTile = 256;
constexpr int kExtendThreads = kTile / 2;  // one double2 column pair per thread
constexpr int kReduceThreads = 256;
constexpr int kSelectThreads = 512;        // selection: one 512-thread block per SM (<= 128 regs for
                                           // the register-resident bounds), few partials and fences
constexpr int kMaxReduceGrid = 2048;       // upper bound of every reduction grid (scratch sizing)
constexpr int kCtaThreads = 256;           // single-CTA GP kernels
constexpr int kMaxRows = 8;                // rows per multi-row extend pass (rebuild)
constexpr int kMaxNmax = 1024;             // largest supported GP training size
constexpr int kMaxDim = 64;                // largest supported search-space dimension
constexpr size_t kCtaSmemLimit = 208 * 1024;  // dynamic staging budget of the single-CTA kernels (their static
                                              // shared arrays need the rest of the 227 KB)

struct KernelParams {
  int nu;
  double lengthscale;
  double s2;  // output variance
};

// Device-resident GP scalars, written by the single-CTA GP kernels.
struct GpScalars {
  double y0;      // shift for the prefix-stable c = L^-1 (y - y0)
  double y_mean;
  double y_std;
  double jitter;
  int32_t n;      // observations in the model
  int32_t status; // 0 ok, 1 pivot <= 0 (factorisation failed), 2 the bordered row taken from the
                  // V column had a pivot below the exactness margin: the exact row is pending
  int32_t fail_row;
  int32_t exact_rows;  // bordered rows that needed the exact substitution after a column attempt
  unsigned long long t[8];  // %globaltimer marks of the last k_gp_append phases (diagnostics)
};

__device__ __forceinline__ unsigned long long gtc_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Device pointers of one GP model.
constexpr int kGpWork = 16;

struct GpDev {
  double* train_x;   // [n_max][d]
  double* train_n2;  // [n_max] squared norms (sequential), for the expansion distance
  double* y;         // [n_max] raw observations
  double* L;         // packed lower factor, row i at i(i+1)/2
  double* c;         // [n_max] L^-1 (y - y0)
  double* e;         // [n_max] L^-1 1
  double* beta;      // [n_max] L^-1 y_standardized
  GpScalars* sc;
  double* scratch;   // [n_max] misc
  int* work;         // [kGpWork] group counters of the persistent rebuild passes
  int n_max;
  int d;
};

struct SpaceDev {
  const double* coords;  // SoA [d][n_pad]
  int64_t n;
  int64_t n_pad;
  int d;
  // Lossless compact copy for the predictive pass (null when some dimension
  // has more than 256 distinct values): coordinate (t, j) is exactly
  // ctab[t * 256 + cidx[t * n_pad + j]] -- 1 byte per value instead of 8.
  const uint8_t* cidx;
  const double* ctab;
};

// Result of the selection kernels (device side, copied to the host).
struct SelectDev {
  int64_t position[3];
  double score[3];
  double lambda;
  double mean_variance;
  double best_std;
  int64_t n_candidates;
  int32_t cv_fallback;
  int32_t gp_status;
  // for cross-shard merging (candidate-axis sharding)
  int64_t best_nonnan_pos[3];
  double best_nonnan_score[3];
  int64_t first_eligible;
  uint32_t first_nan_mask;
  int32_t pad2;
};

struct VarTotals {
  double sum;
  int64_t count;
};

// Deterministic, order-independent total of the posterior variance over the
// unvisited candidates.  Every producer block converts its (block-tree) sum
// to fixed point -- four 42-bit limbs of sum * 2^(120 - ilogb(s2)), exact
// power-of-two scaling, every variance is in [0, s2] -- and adds the limbs
// and its count with integer atomics, so the total does not depend on block
// scheduling and no consumer has to re-reduce per-block partials.
struct VarAccum {
  unsigned long long limb[4];
  unsigned long long count;
  unsigned long long pad[3];
};

// Per-tile summary of the posterior written by every final predictive pass
// (over all candidates of the tile, visited or not): bounds every score in
// the tile, so the selection can skip whole tiles (gtc_kernels.cu k_select).
// var_max < 0 marks a tile without candidates.
struct TileStats {
  double mu_min;
  double var_max;
  double var_min;
  double mu_seed;   // the unvisited candidate with the minimum mean (lowest
  double var_seed;  // position on ties) at pass time: a cheap exact-score seed
  int64_t pos_seed; // -1: none
};

// Where the selection takes the variance total from: an accumulator of this
// run (device), or totals passed by value (candidate-axis sharding).
struct VarSource {
  const VarAccum* acc;
  double s2;
  double sum;
  long long count;
  int direct;
  // candidate-axis sharding: the all-gathered accumulators of every shard
  // ([n_gathered][2] generations); their limbs sum exactly (integers), so the
  // global total is bit-identical to one device holding every tile
  const VarAccum* gathered;
  int n_gathered;
  int gen;
};

// Candidate-axis sharding of the resident loop (gtc_run_attach_comm): every
// shard's selection ends in one record, all-gathered, then merged identically
// on every shard with the reference's best_candidate rule (portfolio.hpp:32-61).
// Record = ShardHdr | x[slots][d] | xfirst[d] | col[slots][n_max] (doubles),
// one slot per acquisition function of the selection mask, in af order: the
// winners' coordinates and V columns, so the shard that does not hold the
// pick can still append its bordered row from the column (column_border_row).
struct ShardHdr {
  int64_t pos[3];     // best non-NaN position per AF slot (global; -1 none)
  double score[3];
  int64_t first;      // lowest eligible global position (-1 none)
  int64_t count;      // eligible candidates of the shard
  uint32_t nan_mask;  // bit af: the first eligible candidate's score is NaN
  int32_t cv_fallback;
  double lambda;
  double mean_var;
  double best_std;
};
__host__ __device__ __forceinline__ int shard_slots(uint32_t mask) {
  return (int)(mask & 1u) + (int)((mask >> 1) & 1u) + (int)((mask >> 2) & 1u);
}
__host__ __device__ __forceinline__ int64_t shard_record_bytes(uint32_t mask, int d, int n_max) {
  const int s = shard_slots(mask);
  return (int64_t)sizeof(ShardHdr) + 8 * ((int64_t)(s + 1) * d + (int64_t)s * n_max);
}

struct LoopDev;

struct SelectParams {
  uint32_t af_mask;
  int lambda_mode;
  double lambda_constant;
  double cv_mu_s;
  double cv_var_s;
  double f_best_raw;
  const int64_t* excluded;  // device, sorted and unique
  int n_excluded;
  int64_t first_eligible;   // host-computed: lowest unvisited, non-excluded position (-1: none)
  int64_t n_candidates;     // host-computed: number of eligible candidates
  LoopDev* loop;            // resident loop: f_best_raw / first_eligible / n_candidates / the
                            // variance total come from the loop state instead, and the
                            // selection's last block advances the loop (loop_advance)
  // resident loop: every block warms L2 with the value-table entry and the V
  // column of its local winners (the last block's lookups and the fused
  // append then hit L2); null outside the loop
  const double* pf_table = nullptr;
  const double* pf_V = nullptr;
  int64_t pf_tile_stride = 0;
  int32_t pf_rows = 0;
  const double* pf_gp[3] = {nullptr, nullptr, nullptr};  // c, e, y: warmed by the last block at its entry (fused append)
  // gtc_observe read-back without a copy engine or a stream synchronisation:
  // the last block also writes the result record and the GP scalars straight
  // into the run's pinned host buffer, then (after a system fence) `seq` into
  // *host_seq, on which the host spins; null: the caller copies them
  SelectDev* host_sel = nullptr;
  GpScalars* host_sc = nullptr;
  uint32_t* host_seq = nullptr;
  uint32_t seq = 0;
};

// Per-block scratch of the selection kernels (sized by reduce_blocks(n)).
struct ReduceBufs {
  double* pvar;        // variance partials (cooperative phase 1)
  long long* pvcnt;
  double* pscore;      // [3 * blocks]
  int64_t* ppos;       // [3 * blocks]
  int64_t* pfirst;
  int32_t* pfinite;    // [blocks] the block's first eligible candidate has finite keys (score not NaN)
  long long* pcnt;
  unsigned int* counter;
  unsigned long long* gthr;  // [3] shared selection thresholds (order-preserving bits; 0 = none)
};

// --- launchers (gtc_kernels.cu); all asynchronous on `stream` -------------

// Single-CTA: factor the Gram matrix of the model's n training points at the
// given jitter (left-looking bordered rows), then c, e, y stats, beta.
void launch_gp_factor(const GpDev& g, KernelParams k, double noise, double jitter, int n,
                      cudaStream_t stream);
// Single-CTA: append observation n0 (coords taken from `space` at `pos`, or
// from `x_explicit` when pos < 0) to the factor; updates scalars and beta.
// Optionally sets the visited bit of `pos`.
// With V (the run's resident V, tile-major) the bordered row is taken from
// candidate pos's V column when its pivot clears the margin (column_border_row).
void launch_gp_append(const GpDev& g, KernelParams k, double noise, const SpaceDev& space,
                      int64_t pos, const double* x_explicit, double y_new, int n0,
                      uint32_t* visited_mark, cudaStream_t stream, const double* V = nullptr,
                      int64_t tile_stride = 0);
// Single-CTA: recompute stats/beta for the prefix of n observations.
void launch_gp_truncate(const GpDev& g, int n, cudaStream_t stream);

// Producer side of a variance total: the final predictive pass (per tile)
// or launch_var_partials add into `acc` (which must be zero) and clear
// `acc_clear` (the next generation's accumulator) -- two generations
// alternate, so no separate zeroing launch is needed.
struct VarPartials {
  const uint32_t* visited;
  VarAccum* acc;
  VarAccum* acc_clear;
};

// Arguments of the kernels that a batch of runs shares one launch of
// (gtc_observe requests gathered across the runs of gtc_run_bo_batch).
struct AppendArgs {
  GpDev g;              // g.L == nullptr: no append for this run in the batch
  KernelParams k;
  double noise;
  SpaceDev sp;
  int64_t pos;
  const double* x_explicit;
  double y_new;
  int n0;
  uint32_t* visited_mark;
  int staged;
  const double* V;      // resident V (tile-major): the bordered row is taken from the observed
  int64_t tile_stride;  // candidate's V column when set (null: exact forward substitution only)
};

struct ExtendArgs {
  SpaceDev sp;
  GpDev g;
  double* V;            // V == nullptr: no pass for this run in the batch
  int64_t tile_stride;
  int n0, r, final_pass, check_status;
  double lengthscale, s2;
  double* mu;
  double* var;
  const uint32_t* visited;  // with acc: per-tile variance totals (final pass)
  VarAccum* acc;
  VarAccum* acc_clear;
  TileStats* tstat;  // final pass: per-tile posterior summary (optional)
  const LoopDev* loop;  // resident loop: n0 and the accumulator generation from the loop state
  int32_t kstar = 0;    // wide rebuild: V rows [n0, n0 + r) already hold the kernel values k(x_t, x) (k_kstar)
};

struct SelectRunArgs {
  const double* mu;
  const double* var;
  const uint32_t* visited;
  int64_t n;
  const GpScalars* sc;
  SelectParams p;
  VarSource vs;
  const TileStats* tstat;
  ReduceBufs b;
  SelectDev* out;       // out == nullptr: no selection for this run in the batch
};

struct GatherDesc {
  const unsigned char* src;
  uint32_t bytes;
  uint32_t dst_offset;
};
struct MarkDesc {
  uint32_t* visited;
  int64_t pos;
  VarAccum* acc;      // optional O(1) update of the variance total
  const double* var;
  double s2;
};
void launch_gather(const GatherDesc* d_descs, int count, unsigned char* dst, cudaStream_t stream);
void launch_mark_batch(const MarkDesc* d_marks, int count, cudaStream_t stream);

AppendArgs make_append_args(const GpDev& g, KernelParams k, double noise, const SpaceDev& space, int64_t pos,
                            const double* x_explicit, double y_new, int n0, uint32_t* visited_mark,
                            size_t* smem_bytes);
ExtendArgs make_pass_args(const SpaceDev& space, const GpDev& g, KernelParams k, double* V, int64_t tile_stride,
                          int n0, double* mu, double* var, const VarPartials* vp, TileStats* tstat);
void launch_gp_append_batch(const AppendArgs* d_args, int count, int nu, size_t smem, cudaStream_t stream);
void launch_extend_batch(const ExtendArgs* d_args, int count, int64_t tiles, int nu, int max_n0, int d,
                         cudaStream_t stream);
void launch_select_batch(const SelectRunArgs* d_args, int count, uint32_t mask, int64_t n, cudaStream_t stream);

// Multi-row V extension over all candidates: rows [n0, n0+r) from rows [0, n0).
// When `final`, also writes the posterior mean/variance of every candidate
// (and, with `vp`, the variance partials).  With `check_status` it is a
// no-op when the preceding bordered row failed.
void launch_extend(const SpaceDev& space, const GpDev& g, KernelParams k, double* V,
                   int64_t tile_stride, int n0, int r, bool final, double* mu, double* var,
                   bool check_status, const VarPartials* vp, TileStats* tstat, cudaStream_t stream);

// Tensor-core V rebuild (k_rebuild): V rows [0, n) of every candidate, bit-identical
// to the streaming k_extend<8> passes; false = not taken (mode off / too large),
// the caller falls back to the streaming passes.  The posterior comes from a
// following final pass (r = 0).
bool launch_rebuild(const SpaceDev& sp, const GpDev& g, KernelParams k, double* V, int64_t tile_stride, int n,
                    cudaStream_t stream);
// Wide streaming rebuild (k_extend_wide: 32 rows per pass, the 8-row panel
// arithmetic): V rows [0, n) and the posterior; false = not taken.
bool launch_rebuild_wide(const SpaceDev& sp, const GpDev& g, KernelParams k, double* V, int64_t tile_stride, int n,
                         double* mu, double* var, const VarPartials* vp, TileStats* tstat, cudaStream_t stream, bool kstar_done = false);
// whether launch_rebuild_wide takes this n (then its kernel values come from launch_kstar)
bool rebuild_wide_taken(const SpaceDev& sp, int n);
void launch_kstar(const SpaceDev& sp, const GpDev& g, KernelParams k, double* V, int64_t tile_stride, int n,
                  cudaStream_t s);
void set_factor_mode(int mode);  // 1 right-looking in shared memory (default), 0 left-looking bordered rows
int factor_mode();
void set_rebuild_mode(int mode);  // 0 streaming 8-row passes, 1 tensor cores, 2 wide 32-row passes (default)
int rebuild_mode();

void launch_var_partials(const double* var, int64_t n, double s2, const VarPartials& vp, cudaStream_t stream);
// Converts a variance source to (sum, count) on the device.
void launch_var_totals(const VarSource& src, VarTotals* out, cudaStream_t stream);

void launch_prior(double* mu, double* var, int64_t n, double s2, TileStats* tstat, cudaStream_t stream);
// Marks/unmarks one candidate; with `acc` (a total valid for the current
// visited set) its variance moves out of / back into the total.
void launch_mark(uint32_t* visited, int64_t pos, int set, cudaStream_t stream, VarAccum* acc = nullptr,
                 const double* var = nullptr, double s2 = 0.0);

// Sum of the variance over unvisited candidates -> totals (deterministic).
void launch_varsum(const double* var, const uint32_t* visited, int64_t n, double* partial_sum,
                   int64_t* partial_cnt, unsigned int* counter, VarTotals* totals,
                   cudaStream_t stream);

// Fused mean-variance (from the partials) + lambda + acquisition + masked
// argmax for every AF in the mask.
void launch_select(const double* mu, const double* var, const uint32_t* visited, int64_t n,
                   const GpScalars* sc, SelectParams p, const VarSource& vs, const TileStats* tstat,
                   const ReduceBufs& bufs, SelectDev* out, cudaStream_t stream, int fused_append_n_max = 0);
// Dynamic shared memory of a loop-mode selection whose last block appends the
// pick (LoopDev::fused_append), for a model of n_max rows.
size_t loop_append_smem(int n_max);

// best_candidate over caller spans of stds (not variances).
void launch_best_candidate(const double* mu, const double* std, const uint8_t* excluded,
                           int64_t n, int af, double best_std, double lambda,
                           const ReduceBufs& bufs, SelectDev* out, cudaStream_t stream);

void launch_scores(const double* mu, const double* sd, int64_t n, int af, double best_std,
                   double lambda, double* out, cudaStream_t stream);

// ---- device search-space enumeration (search_space.hpp:120-166) ----------
// Restriction programs compiled by restriction.cpp (postfix, EnumInstr);
// the kernels evaluate them over the Cartesian grid, then compact the valid
// canonical indices (ascending) with their normalised coordinates.
struct EnumDev {
  const void* code;         // EnumInstr[n_code]
  int n_code;
  const double* values;     // concatenated per-parameter value tables (booleans 0/1, categorical 0)
  const int32_t* val_off;   // [d]
  const uint8_t* str_tab;   // string-comparison tables
  const int32_t* radix;     // [d] values per parameter
  const double* normtab;    // concatenated rank / (k - 1) tables (search_space.hpp:158-166)
  int d;
  int n_values;             // total entries of `values` / `normtab`
  int64_t total;            // Cartesian size (<= 20,000,000)
};
int64_t launch_enumerate_mask(const EnumDev& e, uint32_t* mask, int64_t* block_counts, int64_t* total_valid,
                              cudaStream_t stream);  // returns the number of count blocks
void launch_enumerate_compact(const EnumDev& e, const uint32_t* mask, const int64_t* block_offsets,
                              int64_t n_pad, uint64_t* ids, double* coords, uint8_t* cidx, cudaStream_t stream);

// Initial-sample snap (sampling.hpp:98-117): nearest position of each design
// point (n_pts x d row-major, device); `partial` holds 16 * blocks * n_pts bytes.
int snap_partial_blocks(int64_t n);
void launch_snap(const SpaceDev& sp, const double* pts, int n_pts, void* partial, int64_t* out,
                 cudaStream_t stream);

// ---- resident BO loop (gtc_run_steps) --------------------------------------
// The device-side state of a run's BO loop in simulation mode (objective =
// resident value table): loop_advance turns the last selection into the
// next evaluation -- table lookup, visited mark, candidate count / first
// eligible position, f_best, accumulator generation (loop_advance, run by the
// selection's last block) -- and the append, pass and selection kernels read
// their per-step inputs from here, so a chunk of
// iterations runs without a host round trip (all launch arguments constant).
struct StepRec {  // == gtc_step_record
  int64_t position;
  double value;     // NaN: runtime-invalid
  double lambda;    // exploration factor of the selection that picked it
  int32_t valid;
  int32_t cv_fallback;
  int32_t by;       // acquisition function that produced the pick
  int32_t pad;
};
enum : int32_t { kLoopRunning = 0, kLoopNoCandidates = 1, kLoopPivot = 2, kLoopCapacity = 3 };

// Portfolio state of a multi / advanced-multi run (portfolio.hpp:65-316),
// slots in the fixed order ei, poi, lcb (PortfolioConfig::order).
struct PortDev {
  int32_t mode;            // 0 single AF, 1 multi, 2 advanced multi
  int32_t skip_threshold;
  double discount;
  double rho;              // required improvement
  int32_t active[3];
  int32_t duplicates[3];
  int32_t above[3];
  int32_t below[3];
  double dos[3];           // discounted observation scores
  int64_t last_sug[3];     // most recent suggestion (position; -1 none)
  int64_t cursor;          // rotation cursor
};
struct LoopDev {
  int64_t pos;        // this step's pick
  double y;           // its value
  int32_t valid;
  int32_t n0;         // row of this step's bordered append
  int32_t n;          // observations in the model
  int32_t gen;        // current variance-accumulator generation
  int32_t halt;       // kLoop*
  int32_t step;       // records written
  int32_t af;         // acquisition slot of the strategy
  int32_t n_max;
  int32_t hold;       // steady-state mode: every valid step re-appends at row n0 = hold_n0
  int32_t hold_n0;
  int64_t hold_prev;  // position observed at row hold_n0 (unmarked when replaced), -1 none
  double f_best;      // best valid raw observation (f_best_raw of the selection)
  double f_base;      // hold mode: f_best = min(f_base, y)
  int64_t first;      // lowest unvisited position (-1: none)
  int64_t count;      // unvisited candidates
  int64_t n_space;
  VarAccum* acc;      // [2] the run's accumulator generations
  const double* table;
  uint32_t* visited;
  const double* var;
  double s2;
  const GpScalars* sc;
  const SelectDev* sel;
  StepRec* rec;
  PortDev port;
  double* sorted_y;   // valid observations in ascending order (portfolio median), capacity n_max
  int32_t n_sorted;
  int32_t lambda_mode;  // the selection's exploration parameters (SelectParams in loop mode)
  double lambda_constant;
  double cv_mu_s;
  double cv_var_s;
  // the bordered append of a valid step, run by the selection's last block
  // from the pick's V column (column_border_row)
  GpDev g;
  KernelParams kp;
  double noise;
  SpaceDev sp;
  const double* V;
  int64_t tile_stride;
  int32_t fused_append;     // the selection's last block appends valid picks (loop_append; no append kernel)
  int32_t pad_fa;
  // candidate-axis sharding (nranks > 0): the loop's positions, records and
  // value table are GLOBAL; visited / first / count / acc / var are this
  // shard's candidates [offset, offset + n_space)
  int32_t nranks;
  uint32_t sel_mask;        // the selection's AF mask (record slots)
  int64_t offset;
  unsigned char* send;      // this shard's record (written by k_select's last block)
  const unsigned char* recv;// [nranks] records after the all-gather
  int64_t rec_bytes;
  const VarAccum* gacc;     // [nranks][2] all-gathered accumulators
  double* xrec;             // [step][d] coordinates of each valid step's pick (host replay)
  SelectDev* gsel;          // merged (global) selection
};
// Merge of the all-gathered shard records + loop advance + the bordered row
// of a valid pick from the owning shard's V column (one CTA).
void launch_shard_merge(LoopDev* loop, int nu, int n_max, cudaStream_t stream);
// Loop-mode launch of the single-row pass (args.loop set; args.n0 sized for
// the largest row of the chunk).
// Portfolio script (== gtc_portfolio_op / gtc_portfolio_state).
struct PortOp {
  int32_t kind;  // 0 suggest (picks = per-AF argmax positions), 1 record (af, value)
  int32_t af;
  int64_t picks[3];
  double value;
};
struct PortState {
  int64_t position;
  int32_t by;
  int32_t active[3];
  int32_t duplicates[3];
  int32_t above[3];
  int32_t below[3];
  int32_t pad;
  double dos[3];
};
void launch_portfolio_trace(const PortDev& P, const PortOp* d_ops, int n, PortState* d_out, cudaStream_t stream);
void launch_extend_loop(const ExtendArgs& a, int64_t tiles, int nu, cudaStream_t stream);

// Programmatic dependent launch for this host thread's subsequent launches.
void set_thread_pdl(bool on);

int reduce_blocks(int64_t n);  // grid size used by the reduction kernels
int read_sel_trace(unsigned long long* out, int rows);  // GTC_SEL_TRACE builds (diagnostics)
uint64_t launches();

}  // namespace gtc
