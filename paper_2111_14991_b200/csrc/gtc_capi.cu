// C ABI (include/gridtune_cuda.h) over the sm_100a kernels in gtc_kernels.cu.
//
// Host-side orchestration of the reference's GpModel::fit / predict and the
// run_bo selection step (citations in the header and in gtc_kernels.cu).
// No CPU fallback: every compute path launches device kernels and reports
// GTC_ERR_CUDA when the device is unusable.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <chrono>
#include <cstdlib>
#include <atomic>
#include <semaphore>
#include <thread>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/gridtune_cuda.h"
#include "gtc_comm.hpp"
#include "gtc_internal.h"
#include "restriction.hpp"

using namespace gtc;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define GTC_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) return fail(GTC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define GTC_LAUNCHED()                                                                   \
  do {                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess) return fail(GTC_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
int dalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * count);
  if (e != cudaSuccess) {
    *p = nullptr;
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? GTC_ERR_OOM : GTC_ERR_CUDA,
                std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  return GTC_OK;
}

int64_t pad_tiles(int64_t n) { return ((n + kTile - 1) / kTile) * kTile; }
size_t packed_size(int n) { return (size_t)n * (size_t)(n + 1) / 2; }

int check_kernel(const gtc_kernel* k) {
  if (!k) return fail(GTC_ERR_INVALID, "kernel is null");
  if (k->nu < 0 || k->nu > 2) return fail(GTC_ERR_INVALID, "unknown Matern nu");
  // MaternKernel constructor checks, gp.hpp:33-37
  if (!(k->lengthscale > 0.0)) return fail(GTC_ERR_INVALID, "kernel lengthscale must be positive");
  if (!(k->output_variance > 0.0)) return fail(GTC_ERR_INVALID, "kernel output variance must be positive");
  return GTC_OK;
}

KernelParams kparams(const gtc_kernel& k) { return KernelParams{k.nu, k.lengthscale, k.output_variance}; }

std::string fmt_jitter(double j) { return std::to_string(j); }  // std::to_string as gp.hpp:126

// Scratch of the multi-block reductions (sized for reduce_blocks()).
struct ReduceScratch {
  ReduceBufs b{};
  double* vsum = nullptr;      // k_varsum partials
  int64_t* vcnt = nullptr;
  unsigned int* vcounter = nullptr;
  VarTotals* totals = nullptr;
  SelectDev* sel = nullptr;
  SelectDev* h_sel = nullptr;  // pinned
  VarTotals* h_totals = nullptr;

  int init(int64_t n) {
    const int nb = std::max(reduce_blocks(n), kMaxReduceGrid);  // covers the selection grid too
    int rc;
    if ((rc = dalloc(&b.pvar, nb)) || (rc = dalloc(&b.pvcnt, nb)) || (rc = dalloc(&b.pscore, 3 * nb)) ||
        (rc = dalloc(&b.ppos, 3 * nb)) || (rc = dalloc(&b.pfirst, nb)) || (rc = dalloc(&b.pfinite, nb)) || (rc = dalloc(&b.pcnt, nb)) ||
        (rc = dalloc(&b.counter, 1)) || (rc = dalloc(&b.gthr, 3)) || (rc = dalloc(&vsum, nb)) || (rc = dalloc(&vcnt, nb)) ||
        (rc = dalloc(&vcounter, 1)) || (rc = dalloc(&totals, 1)) || (rc = dalloc(&sel, 1)))
      return rc;
    GTC_CUDA(cudaMemset(b.counter, 0, sizeof(unsigned int)));
    GTC_CUDA(cudaMemset(b.gthr, 0, 3 * sizeof(unsigned long long)));
    GTC_CUDA(cudaMemset(vcounter, 0, sizeof(unsigned int)));
    GTC_CUDA(cudaMallocHost(&h_sel, sizeof(SelectDev)));
    GTC_CUDA(cudaMallocHost(&h_totals, sizeof(VarTotals)));
    return GTC_OK;
  }
  void release() {
    cudaFree(b.pvar); cudaFree(b.pvcnt); cudaFree(b.pscore); cudaFree(b.ppos); cudaFree(b.pfirst); cudaFree(b.pfinite);
    cudaFree(b.pcnt); cudaFree(b.counter); cudaFree(b.gthr); cudaFree(vsum); cudaFree(vcnt); cudaFree(vcounter);
    cudaFree(totals); cudaFree(sel);
    if (h_sel) cudaFreeHost(h_sel);
    if (h_totals) cudaFreeHost(h_totals);
  }
};

// Device GP model storage.
struct GpStore {
  GpDev dev{};
  GpScalars* h_sc = nullptr;  // pinned
  int init(int n_max, int d) {
    int rc;
    dev.n_max = n_max;
    dev.d = d;
    if ((rc = dalloc(&dev.train_x, (size_t)n_max * d)) || (rc = dalloc(&dev.train_n2, n_max)) ||
        (rc = dalloc(&dev.y, n_max)) || (rc = dalloc(&dev.L, packed_size(n_max) + 2)) ||
        (rc = dalloc(&dev.c, n_max)) || (rc = dalloc(&dev.e, n_max)) ||
        (rc = dalloc(&dev.beta, n_max)) || (rc = dalloc(&dev.sc, 1)) ||
        (rc = dalloc(&dev.scratch, n_max)) || (rc = dalloc(&dev.work, kGpWork)))
      return rc;
    GTC_CUDA(cudaMemset(dev.sc, 0, sizeof(GpScalars)));
    GTC_CUDA(cudaMallocHost(&h_sc, sizeof(GpScalars)));
    std::memset(h_sc, 0, sizeof(GpScalars));
    h_sc->y_std = 1.0;
    return GTC_OK;
  }
  void release() {
    cudaFree(dev.train_x); cudaFree(dev.train_n2); cudaFree(dev.y); cudaFree(dev.L);
    cudaFree(dev.c); cudaFree(dev.e); cudaFree(dev.beta); cudaFree(dev.sc); cudaFree(dev.scratch); cudaFree(dev.work);
    if (h_sc) cudaFreeHost(h_sc);
  }
};

// Factorises the n training points already on the device with the
// reference's jitter escalation (gp.hpp:116-129), starting at `start_jitter`
// and never exceeding base * 2^6.  On success h_sc holds the scalars.
int factor_with_escalation(GpStore& gp, const gtc_kernel& k, double noise, double base_jitter,
                           double start_jitter, int n, cudaStream_t s,
                           const std::function<int()>& after_first_launch = {}) {
  double jitter = start_jitter;
  // attempts already "spent" below start_jitter (each failed in the reference)
  int attempts = 0;
  for (double j = base_jitter; j < start_jitter; j *= 2.0) ++attempts;
  if (attempts > 6) {
    return fail(GTC_ERR_CONDITIONING, "Gram matrix factorization failed after jitter escalation to " +
                                          fmt_jitter(base_jitter * 64.0));
  }
  for (bool first = true;; first = false) {
    launch_gp_factor(gp.dev, kparams(k), noise, jitter, n, s);
    GTC_LAUNCHED();
    if (first && after_first_launch) {
      const int rc = after_first_launch();
      if (rc) return rc;
    }
    GTC_CUDA(cudaMemcpyAsync(gp.h_sc, gp.dev.sc, sizeof(GpScalars), cudaMemcpyDeviceToHost, s));
    GTC_CUDA(cudaStreamSynchronize(s));
    if (gp.h_sc->status == 0) return GTC_OK;
    if (++attempts > 6) {
      return fail(GTC_ERR_CONDITIONING,
                  "Gram matrix factorization failed after jitter escalation to " + fmt_jitter(jitter));
    }
    jitter *= 2.0;
  }
}

// Rebuilds V rows [0, n) for `space` (chunks of kMaxRows) and the posterior.
int rebuild_predictions(const SpaceDev& sp, GpStore& gp, const gtc_kernel& k, double* V,
                        int64_t tile_stride, int n, double* mu, double* var, const VarPartials* vp,
                        TileStats* tstat, cudaStream_t s, bool kstar_done = false) {
  if (n == 0) {
    launch_prior(mu, var, sp.n_pad, k.output_variance, tstat, s);
    GTC_LAUNCHED();
    return GTC_OK;
  }
  if (launch_rebuild_wide(sp, gp.dev, kparams(k), V, tile_stride, n, mu, var, vp, tstat, s, kstar_done)) {
    GTC_LAUNCHED();
    return GTC_OK;
  }
  if (launch_rebuild(sp, gp.dev, kparams(k), V, tile_stride, n, s)) {
    GTC_LAUNCHED();
    // posterior, tile summaries and variance total from the rebuilt rows
    launch_extend(sp, gp.dev, kparams(k), V, tile_stride, n, 0, true, mu, var, false, vp, tstat, s);
    GTC_LAUNCHED();
    return GTC_OK;
  }
  for (int n0 = 0; n0 < n; n0 += kMaxRows) {
    const int r = std::min(kMaxRows, n - n0);
    launch_extend(sp, gp.dev, kparams(k), V, tile_stride, n0, r, n0 + r == n, mu, var, false, vp, tstat, s);
    GTC_LAUNCHED();
  }
  return GTC_OK;
}

void fill_info(gtc_fit_info* info, const GpScalars& sc, int n, int rebuilt) {
  if (!info) return;
  info->n = n;
  info->rebuilt = rebuilt;
  info->y_mean = sc.y_mean;
  info->y_std = sc.y_std;
  info->jitter = sc.jitter;
}

int check_fit_inputs(const double* y, int n, double noise, double jitter) {
  if (n < 0) return fail(GTC_ERR_INVALID, "GP fit: observation count does not match input count");
  if (!(noise >= 0.0)) return fail(GTC_ERR_INVALID, "GP fit: noise must be non-negative");
  if (!(jitter > 0.0)) return fail(GTC_ERR_INVALID, "GP fit: jitter must be positive");
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(y[i])) return fail(GTC_ERR_INVALID, "GP fit: observations must be finite");
  return GTC_OK;
}

void copy_result(const SelectDev& s, gtc_select_result* out) {
  for (int k = 0; k < 3; ++k) {
    out->position[k] = s.position[k];
    out->score[k] = s.score[k];
  }
  out->lambda = s.lambda;
  out->mean_variance = s.mean_variance;
  out->best_std = s.best_std;
  out->n_candidates = s.n_candidates;
  out->cv_fallback = s.cv_fallback;
}

}  // namespace

// =============================================================== handles

struct gtc_space {
  int device = 0;
  int64_t n = 0, n_pad = 0;
  int d = 0;
  double* coords = nullptr;          // device SoA [d][n_pad]
  uint8_t* cidx = nullptr;           // device [d][n_pad] value indices (SpaceDev), or null
  double* ctab = nullptr;            // device [d][256] distinct values per dimension
  std::vector<double> host_coords;   // row-major n x d (gathers for fit)
  std::vector<uint64_t> ids;         // canonical indices (enumerated spaces)
  uint64_t cartesian = 0;            // Cartesian size (enumerated spaces)
  // idle run handles (gtc_run_release): reused by gtc_run_acquire, so sweeps
  // of many runs allocate device memory once per concurrent run, not per run
  std::mutex pool_mu;
  std::vector<gtc_run*> pool;
  SpaceDev dev() const { return SpaceDev{coords, n, n_pad, d, cidx, ctab}; }
};

struct gtc_run {
  gtc_space* space = nullptr;
  gtc_group* group = nullptr;  // batched observe (gtc_run_set_group)
  gtc_model_config cfg{};
  cudaStream_t stream = nullptr;
  GpStore gp;
  ReduceScratch red;
  double* V = nullptr;
  int64_t tile_stride = 0;
  double* mu = nullptr;
  double* var = nullptr;
  uint32_t* visited = nullptr;
  int64_t* excluded = nullptr;
  int excluded_cap = 0;
  std::vector<int64_t> ex_host;  // last selection's exclusions (sorted, unique)
  int64_t first_hint = 0;        // <= the lowest unvisited position
  std::vector<uint32_t> visited_host;
  int64_t visited_count = 0;
  int n = 0;
  double jitter = 0.0;
  bool predictions_valid = false;
  std::vector<double> y_host;
  std::vector<double> x_host;  // n x d training coordinates
  // candidate-axis sharding: this run's candidates are global positions
  // [shard_offset, shard_offset + space->n)
  int64_t shard_offset = 0;
  // device-resident sharding of the resident loop (gtc_run_attach_comm)
  gtc_comm* comm = nullptr;
  int64_t n_global = 0;
  unsigned char* d_send = nullptr;  // this shard's selection record
  unsigned char* d_recv = nullptr;  // [nranks] gathered records
  VarAccum* d_gacc = nullptr;       // [nranks][2] gathered accumulators
  double* d_xrec = nullptr;         // [rec_cap][d] pick coordinates per step
  int xrec_cap = 0;
  std::vector<double> xrec_host;
  double* d_xnew = nullptr;       // device copy of an explicit new point (d doubles)
  double* h_xnew = nullptr;       // pinned staging
  struct Readback {
    SelectDev sel;
    GpScalars sc;
    uint32_t seq;  // written last by the selection's last block (direct read-back)
    uint32_t pad;
  };
  Readback* h_rb = nullptr;  // pinned: the selection writes its result here directly (gtc_observe)
  uint32_t rb_seq = 0;
  // fixed-point variance totals over the unvisited candidates, two
  // alternating generations (VarAccum); acc_valid: the current generation
  // matches the current visited set and predictions
  TileStats* tstat = nullptr;  // [tiles] posterior summary per tile (selection pruning)
  // gtc_truncate without `info` defers the standardisation / beta of the
  // prefix (k_gp_truncate) to its first consumer; a bordered append
  // recomputes them anyway (-1: up to date)
  int stats_stale = -1;
  VarAccum* acc = nullptr;  // [2]
  int acc_gen = 0;
  bool acc_valid = false;
  int tiles = 0;
  // producer side of the next generation (becomes current)
  VarPartials vp() {
    acc_gen ^= 1;
    return VarPartials{visited, acc + acc_gen, acc + (acc_gen ^ 1)};
  }
  VarSource vsrc() const { return VarSource{acc + acc_gen, cfg.kernel.output_variance, 0.0, 0, 0}; }
  // the total to update in O(1) on a mark, when it matches the visited set
  VarAccum* live_acc() const { return acc_valid && predictions_valid ? acc + acc_gen : nullptr; }
  // resident loop (gtc_run_steps): value table, loop state, step records
  double* d_values = nullptr;
  int64_t values_cap = 0;
  bool has_values = false;
  LoopDev* d_loop = nullptr;
  LoopDev* h_loop = nullptr;  // pinned
  StepRec* d_rec = nullptr;
  int rec_cap = 0;
  std::vector<cudaEvent_t> step_events;  // GTC_STEPS_TIMING: 3 per step + 1
  bool pdl = true;                       // programmatic dependent launch (gtc_run_set_pdl)
  PortDev port{};                        // portfolio state between gtc_run_steps calls (mode 0: none)
  // gtc_run_steps without PDL: captured iteration graphs (kSteps iterations and
  // one iteration), reused while their launch arguments are unchanged
  struct StepGraphs {
    std::string key;
    cudaGraphExec_t many = nullptr, one = nullptr;
    bool failed = false;
    void release() {
      if (many) cudaGraphExecDestroy(many);
      if (one) cudaGraphExecDestroy(one);
      many = one = nullptr;
      key.clear();
    }
  } graphs;
  std::vector<double> sorted_host;
  double* d_sorted_y = nullptr;          // [n_max] sorted valid observations (portfolio median)
  int timed_steps = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;          // last predictive pass
  cudaEvent_t ev_step0 = nullptr, ev_step1 = nullptr;  // last gtc_observe device span
  bool pass_timed = false, step_timed = false, step_appended = false;
  // full fits: the kernel values run on `side` beside the factorisation
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

struct gtc_gp {
  int device = 0;
  gtc_kernel kernel{};
  double noise = 0, jitter = 0;
  int n = 0, d = 0;
  cudaStream_t stream = nullptr;
  GpStore gp;
};

// =============================================================== library

extern "C" const char* gtc_last_error(void) { return g_last_error.c_str(); }
extern "C" void gtc_internal_set_error(const char* msg) { g_last_error = msg ? msg : ""; }
extern "C" const char* gtc_version(void) { return "gridtune-b200 0.2 (sm_100a)"; }
extern "C" uint64_t gtc_kernel_launches(void) { return launches(); }

// =============================================================== space

// Discrete search spaces have few distinct values per parameter (the
// normalised ranks, search_space.hpp:158-166): when every dimension has at
// most 256, the pass reads 1-byte indices into exact per-dimension tables
// (bit patterns are kept, so the coordinates are reproduced exactly).
static cudaError_t compress_coords(gtc_space* s, const std::vector<double>& soa) {
  std::vector<uint8_t> idx((size_t)s->d * s->n_pad, 0);
  std::vector<double> tab((size_t)s->d * 256, 0.0);
  for (int t = 0; t < s->d; ++t) {
    std::unordered_map<uint64_t, int> slot;
    for (int64_t j = 0; j < s->n; ++j) {
      const double v = soa[(size_t)t * s->n_pad + j];
      uint64_t bits;
      std::memcpy(&bits, &v, sizeof bits);
      auto it = slot.find(bits);
      if (it == slot.end()) {
        if (slot.size() == 256) return cudaSuccess;  // not compressible: the pass reads coords
        it = slot.emplace(bits, (int)slot.size()).first;
        tab[(size_t)t * 256 + it->second] = v;
      }
      idx[(size_t)t * s->n_pad + j] = (uint8_t)it->second;
    }
  }
  cudaError_t e = cudaMalloc(&s->cidx, idx.size());
  if (e == cudaSuccess) e = cudaMalloc(&s->ctab, tab.size() * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(s->cidx, idx.data(), idx.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(s->ctab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice);
  return e;
}

extern "C" int gtc_space_create(int device, const double* coords, int64_t n, int32_t d,
                                gtc_space** out) {
  if (!out) return fail(GTC_ERR_INVALID, "out is null");
  *out = nullptr;
  if (n <= 0) return fail(GTC_ERR_INVALID, "search space has no configurations");
  if (d <= 0 || d > kMaxDim) return fail(GTC_ERR_INVALID, "search-space dimension out of range [1, 64]");
  if (!coords) return fail(GTC_ERR_INVALID, "coords is null");
  GTC_CUDA(cudaSetDevice(device));
  auto* s = new gtc_space();
  s->device = device;
  s->n = n;
  s->n_pad = pad_tiles(n);
  s->d = d;
  s->host_coords.assign(coords, coords + n * d);
  std::vector<double> soa((size_t)d * s->n_pad, 0.0);
  for (int64_t j = 0; j < n; ++j)
    for (int t = 0; t < d; ++t) soa[(size_t)t * s->n_pad + j] = coords[j * d + t];
  int rc = dalloc(&s->coords, soa.size());
  if (rc) {
    delete s;
    return rc;
  }
  cudaError_t e = cudaMemcpy(s->coords, soa.data(), soa.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = compress_coords(s, soa);
  if (e != cudaSuccess) {
    gtc_space_destroy(s);
    return fail(GTC_ERR_CUDA, std::string("space upload: ") + cudaGetErrorString(e));
  }
  *out = s;
  return GTC_OK;
}

extern "C" int gtc_space_destroy(gtc_space* s) {
  if (!s) return GTC_OK;
  std::vector<gtc_run*> idle;
  {
    std::lock_guard<std::mutex> lk(s->pool_mu);
    idle.swap(s->pool);
  }
  for (gtc_run* r : idle) gtc_run_destroy(r);
  cudaSetDevice(s->device);
  cudaFree(s->coords);
  cudaFree(s->cidx);
  cudaFree(s->ctab);
  delete s;
  return GTC_OK;
}

extern "C" int64_t gtc_space_size(const gtc_space* s) { return s ? s->n : -1; }

// =============================================================== enumeration

static int convert_params(const gtc_param_def* params, int32_t n_params, std::vector<ParamDef>* out) {
  if (n_params < 0 || (n_params > 0 && !params)) return fail(GTC_ERR_INVALID, "params is null");
  out->clear();
  for (int32_t i = 0; i < n_params; ++i) {
    const gtc_param_def& g = params[i];
    ParamDef p;
    p.name = g.name ? g.name : "";
    if (g.kind < 0 || g.kind > 2) return fail(GTC_ERR_INVALID, "parameter '" + p.name + "' has an unknown kind");
    if (g.n_values < 0) return fail(GTC_ERR_INVALID, "parameter '" + p.name + "' has a negative value count");
    p.kind = static_cast<ParamKind>(g.kind);
    for (int32_t v = 0; v < g.n_values; ++v) {
      if (p.kind == ParamKind::numeric) {
        if (!g.numbers) return fail(GTC_ERR_INVALID, "parameter '" + p.name + "' numbers is null");
        p.numbers.push_back(g.numbers[v]);
      } else if (p.kind == ParamKind::categorical) {
        if (!g.strings || !g.strings[v]) return fail(GTC_ERR_INVALID, "parameter '" + p.name + "' strings is null");
        p.strings.emplace_back(g.strings[v]);
      } else {
        if (!g.booleans) return fail(GTC_ERR_INVALID, "parameter '" + p.name + "' booleans is null");
        p.booleans.push_back(g.booleans[v] != 0);
      }
    }
    out->push_back(std::move(p));
  }
  return GTC_OK;
}

extern "C" int gtc_restriction_validate(const gtc_param_def* params, int32_t n_params, const char* text,
                                        int64_t* error_position) {
  std::vector<ParamDef> ps;
  int rc = convert_params(params, n_params, &ps);
  if (rc) return rc;
  EnumProgram prog;
  RestrictionError err;
  if (!compile_restriction(text ? text : "", ps, &prog, &err)) {
    if (error_position) *error_position = (int64_t)err.position;
    return fail(err.parse ? GTC_ERR_PARSE : GTC_ERR_INVALID, err.message);
  }
  return GTC_OK;
}

// RAII for the enumeration's temporary device buffers
// Temporary device buffers of one call, stream-ordered (cudaMallocAsync /
// cudaFreeAsync from the device's pool): unlike cudaFree, releasing them does
// not synchronise the whole device, so concurrent runs' pipelines keep going.
struct DevBufs {
  cudaStream_t stream;
  std::vector<void*> ptrs;
  explicit DevBufs(cudaStream_t s) : stream(s) {}
  ~DevBufs() {
    for (void* p : ptrs) cudaFreeAsync(p, stream);
  }
  template <class T>
  int get(T** p, size_t count) {
    if (count == 0) count = 1;
    const cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), sizeof(T) * count, stream);
    if (e != cudaSuccess) {
      *p = nullptr;
      cudaGetLastError();
      return fail(e == cudaErrorMemoryAllocation ? GTC_ERR_OOM : GTC_ERR_CUDA,
                  std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
    }
    ptrs.push_back(*p);
    return GTC_OK;
  }
};

extern "C" int gtc_space_enumerate(int device, const gtc_param_def* params, int32_t n_params,
                                   const char* const* restrictions, int32_t n_restrictions,
                                   int64_t* error_position, gtc_space** out) {
  if (!out) return fail(GTC_ERR_INVALID, "out is null");
  *out = nullptr;
  std::vector<ParamDef> ps;
  int rc = convert_params(params, n_params, &ps);
  if (rc) return rc;
  // SearchSpace(params, sources): every restriction is parsed, then the
  // parameters are validated (search_space.hpp:35-44)
  EnumProgram prog;
  for (int32_t r = 0; r < n_restrictions; ++r) {
    RestrictionError err;
    if (!compile_restriction(restrictions && restrictions[r] ? restrictions[r] : "", ps, &prog, &err)) {
      if (error_position) *error_position = (int64_t)err.position;
      return fail(err.parse ? GTC_ERR_PARSE : GTC_ERR_INVALID, err.message);
    }
  }
  {
    RestrictionError err;
    if (!validate_params(ps, &err)) return fail(GTC_ERR_INVALID, err.message);
  }
  const int d = (int)ps.size();
  if (d > kMaxDim) return fail(GTC_ERR_INVALID, "search-space dimension out of range [1, 64]");
  // cartesian_size() and the enumeration limit (search_space.hpp:120-127)
  constexpr uint64_t kEnumerationLimit = 20000000ull;
  uint64_t total = 1;
  bool over = false;
  for (const ParamDef& p : ps) {
    if (total > (~0ull) / p.size()) over = true;
    total *= p.size();
  }
  if (over || total > kEnumerationLimit)
    return fail(GTC_ERR_INVALID, "Cartesian size " + std::to_string(total) + " exceeds the enumeration limit of " +
                                     std::to_string(kEnumerationLimit));
  // value tables (booleans 0/1), radices, exact normalised coordinates
  std::vector<double> values, normtab;
  std::vector<int32_t> val_off, radix;
  bool compressible = true;
  for (const ParamDef& p : ps) {
    const size_t k = p.size();
    val_off.push_back((int32_t)values.size());
    radix.push_back((int32_t)k);
    compressible = compressible && k <= 256;
    for (size_t r = 0; r < k; ++r) {
      values.push_back(p.kind == ParamKind::numeric ? p.numbers[r]
                       : p.kind == ParamKind::boolean ? (p.booleans[r] ? 1.0 : 0.0) : 0.0);
      normtab.push_back(k <= 1 ? 0.0 : static_cast<double>(r) / static_cast<double>(k - 1));
    }
  }
  if (values.size() > 4096) return fail(GTC_ERR_INVALID, "more than 4096 parameter values in total");
  GTC_CUDA(cudaSetDevice(device));
  cudaStream_t st;
  GTC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{st};
  DevBufs tmp(st);
  EnumInstr* d_code;
  double *d_values, *d_norm;
  int32_t *d_off, *d_radix;
  uint8_t* d_str;
  uint32_t* d_mask;
  int64_t *d_counts, *d_total;
  const int64_t words = (int64_t)((total + 31) / 32);
  if ((rc = tmp.get(&d_code, prog.code.size())) || (rc = tmp.get(&d_values, values.size())) ||
      (rc = tmp.get(&d_norm, normtab.size())) || (rc = tmp.get(&d_off, d)) || (rc = tmp.get(&d_radix, d)) ||
      (rc = tmp.get(&d_str, std::max<size_t>(prog.str_tables.size(), 1))) || (rc = tmp.get(&d_mask, words)) ||
      (rc = tmp.get(&d_counts, 2048)) || (rc = tmp.get(&d_total, 1)))
    return rc;
  GTC_CUDA(cudaMemcpyAsync(d_code, prog.code.data(), sizeof(EnumInstr) * prog.code.size(), cudaMemcpyHostToDevice, st));
  GTC_CUDA(cudaMemcpyAsync(d_values, values.data(), sizeof(double) * values.size(), cudaMemcpyHostToDevice, st));
  GTC_CUDA(cudaMemcpyAsync(d_norm, normtab.data(), sizeof(double) * normtab.size(), cudaMemcpyHostToDevice, st));
  GTC_CUDA(cudaMemcpyAsync(d_off, val_off.data(), sizeof(int32_t) * d, cudaMemcpyHostToDevice, st));
  GTC_CUDA(cudaMemcpyAsync(d_radix, radix.data(), sizeof(int32_t) * d, cudaMemcpyHostToDevice, st));
  if (!prog.str_tables.empty())
    GTC_CUDA(cudaMemcpyAsync(d_str, prog.str_tables.data(), prog.str_tables.size(), cudaMemcpyHostToDevice, st));
  const EnumDev e{d_code, (int)prog.code.size(), d_values, d_off, d_str, d_radix, d_norm, d, (int)values.size(),
                  (int64_t)total};
  launch_enumerate_mask(e, d_mask, d_counts, d_total, st);
  GTC_LAUNCHED();
  int64_t n = 0;
  GTC_CUDA(cudaMemcpyAsync(&n, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GTC_CUDA(cudaStreamSynchronize(st));
  if (n == 0) return fail(GTC_ERR_EMPTY, "restrictions exclude every configuration");
  auto* s = new gtc_space();
  s->device = device;
  s->n = n;
  s->n_pad = pad_tiles(n);
  s->d = d;
  s->cartesian = total;
  uint64_t* d_ids;
  if ((rc = tmp.get(&d_ids, n)) || (rc = dalloc(&s->coords, (size_t)d * s->n_pad)) ||
      (compressible && ((rc = dalloc(&s->cidx, (size_t)d * s->n_pad)) || (rc = dalloc(&s->ctab, (size_t)d * 256))))) {
    gtc_space_destroy(s);
    return rc;
  }
  cudaError_t ce = cudaMemsetAsync(s->coords, 0, sizeof(double) * d * s->n_pad, st);
  if (ce == cudaSuccess && compressible) ce = cudaMemsetAsync(s->cidx, 0, (size_t)d * s->n_pad, st);
  if (ce == cudaSuccess && compressible) {
    std::vector<double> ctab((size_t)d * 256, 0.0);
    for (int t = 0; t < d; ++t)
      for (int r = 0; r < radix[t]; ++r) ctab[(size_t)t * 256 + r] = normtab[val_off[t] + r];
    ce = cudaMemcpy(s->ctab, ctab.data(), ctab.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  if (ce != cudaSuccess) {
    gtc_space_destroy(s);
    return fail(GTC_ERR_CUDA, std::string("enumerate: ") + cudaGetErrorString(ce));
  }
  launch_enumerate_compact(e, d_mask, d_counts, s->n_pad, d_ids, s->coords, s->cidx, st);
  ce = cudaGetLastError();
  std::vector<double> soa((size_t)d * s->n_pad);
  s->ids.resize(n);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(s->ids.data(), d_ids, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(soa.data(), s->coords, sizeof(double) * soa.size(), cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) {
    gtc_space_destroy(s);
    return fail(GTC_ERR_CUDA, std::string("enumerate: ") + cudaGetErrorString(ce));
  }
  s->host_coords.resize((size_t)n * d);  // row-major host view (fit gathers)
  for (int64_t j = 0; j < n; ++j)
    for (int t = 0; t < d; ++t) s->host_coords[(size_t)j * d + t] = soa[(size_t)t * s->n_pad + j];
  *out = s;
  return GTC_OK;
}

extern "C" int gtc_space_ids(const gtc_space* s, uint64_t* ids) {
  if (!s || !ids) return fail(GTC_ERR_INVALID, "null argument");
  if (s->ids.empty()) return fail(GTC_ERR_INVALID, "space was not enumerated: no canonical ids");
  std::memcpy(ids, s->ids.data(), sizeof(uint64_t) * s->ids.size());
  return GTC_OK;
}

extern "C" uint64_t gtc_space_cartesian_size(const gtc_space* s) { return s ? s->cartesian : 0; }

extern "C" int gtc_space_nearest(const gtc_space* s, const double* points, int32_t n, int64_t* positions) {
  if (!s || !positions || (n > 0 && !points)) return fail(GTC_ERR_INVALID, "null argument");
  if (n <= 0) return GTC_OK;
  GTC_CUDA(cudaSetDevice(s->device));
  cudaStream_t st;
  GTC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{st};
  DevBufs tmp(st);
  double* d_pts;
  unsigned char* d_part;
  int64_t* d_out;
  const int blocks = snap_partial_blocks(s->n);
  int rc;
  if ((rc = tmp.get(&d_pts, (size_t)n * s->d)) || (rc = tmp.get(&d_part, (size_t)16 * blocks * n)) ||
      (rc = tmp.get(&d_out, n)))
    return rc;
  GTC_CUDA(cudaMemcpyAsync(d_pts, points, sizeof(double) * n * s->d, cudaMemcpyHostToDevice, st));
  launch_snap(s->dev(), d_pts, n, d_part, d_out, st);
  GTC_LAUNCHED();
  GTC_CUDA(cudaMemcpyAsync(positions, d_out, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
  GTC_CUDA(cudaStreamSynchronize(st));
  return GTC_OK;
}
extern "C" const double* gtc_space_coords(const gtc_space* s) { return s ? s->host_coords.data() : nullptr; }
extern "C" int32_t gtc_space_dimension(const gtc_space* s) { return s ? s->d : -1; }
extern "C" int32_t gtc_space_device(const gtc_space* s) { return s ? s->device : -1; }

// =============================================================== run

extern "C" int gtc_run_destroy(gtc_run* r) {
  if (!r) return GTC_OK;
  cudaSetDevice(r->space->device);
  if (r->stream) cudaStreamSynchronize(r->stream);
  r->gp.release();
  r->red.release();
  cudaFree(r->V);
  cudaFree(r->mu);
  cudaFree(r->var);
  cudaFree(r->visited);
  cudaFree(r->excluded);
  cudaFree(r->acc);
  cudaFree(r->tstat);
  cudaFree(r->d_xnew);
  cudaFree(r->d_values);
  cudaFree(r->d_loop);
  cudaFree(r->d_rec);
  cudaFree(r->d_sorted_y);
  cudaFree(r->d_send);
  cudaFree(r->d_recv);
  cudaFree(r->d_gacc);
  cudaFree(r->d_xrec);
  if (r->h_loop) cudaFreeHost(r->h_loop);
  for (cudaEvent_t ev : r->step_events) cudaEventDestroy(ev);
  r->graphs.release();
  if (r->h_xnew) cudaFreeHost(r->h_xnew);
  if (r->h_rb) cudaFreeHost(r->h_rb);
  for (cudaEvent_t ev : {r->ev0, r->ev1, r->ev_step0, r->ev_step1, r->ev_fork, r->ev_join})
    if (ev) cudaEventDestroy(ev);
  if (r->side) cudaStreamDestroy(r->side);
  if (r->stream) cudaStreamDestroy(r->stream);
  delete r;
  return GTC_OK;
}

extern "C" int gtc_run_create(gtc_space* space, const gtc_model_config* cfg, gtc_run** out) {
  if (!out) return fail(GTC_ERR_INVALID, "out is null");
  *out = nullptr;
  if (!space || !cfg) return fail(GTC_ERR_INVALID, "space/config is null");
  int rc = check_kernel(&cfg->kernel);
  if (rc) return rc;
  if (!(cfg->noise >= 0.0)) return fail(GTC_ERR_INVALID, "GP fit: noise must be non-negative");
  if (!(cfg->jitter > 0.0)) return fail(GTC_ERR_INVALID, "GP fit: jitter must be positive");
  if (cfg->n_max < 1 || cfg->n_max > kMaxNmax)
    return fail(GTC_ERR_CONFIG, "n_max out of range [1, 1024]");
  GTC_CUDA(cudaSetDevice(space->device));
  auto* r = new gtc_run();
  r->space = space;
  r->cfg = *cfg;
  r->jitter = cfg->jitter;
  r->tile_stride = (int64_t)cfg->n_max * kTile;
  const int64_t tiles = space->n_pad / kTile;
  const int64_t words = (space->n + 31) / 32;
  if ((rc = r->gp.init(cfg->n_max, space->d)) || (rc = r->red.init(space->n)) ||
      (rc = dalloc(&r->V, (size_t)tiles * r->tile_stride)) || (rc = dalloc(&r->mu, space->n_pad)) ||
      (rc = dalloc(&r->var, space->n_pad)) || (rc = dalloc(&r->visited, words)) ||
      (rc = dalloc(&r->acc, 2)) || (rc = dalloc(&r->tstat, tiles))) {
    gtc_run_destroy(r);
    return rc;
  }
  cudaError_t e = cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r->side, cudaStreamNonBlocking);
  for (cudaEvent_t* ev : {&r->ev0, &r->ev1, &r->ev_step0, &r->ev_step1})
    if (e == cudaSuccess) e = cudaEventCreate(ev);
  for (cudaEvent_t* ev : {&r->ev_fork, &r->ev_join})
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMemset(r->visited, 0, words * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(r->acc, 0, 2 * sizeof(VarAccum));
  if (e == cudaSuccess) e = cudaMallocHost(&r->h_rb, sizeof(gtc_run::Readback));
  if (e == cudaSuccess) std::memset(r->h_rb, 0, sizeof(gtc_run::Readback));  // (seq starts at 0)
  if (e == cudaSuccess) e = cudaMallocHost(&r->h_xnew, sizeof(double) * kMaxDim);
  if (e == cudaSuccess) e = cudaMalloc(&r->d_xnew, sizeof(double) * kMaxDim);
  if (e != cudaSuccess) {
    gtc_run_destroy(r);
    return fail(GTC_ERR_CUDA, std::string("run create: ") + cudaGetErrorString(e));
  }
  r->visited_host.assign(words, 0u);
  r->tiles = (int)tiles;
  *out = r;
  return GTC_OK;
}

extern "C" int gtc_run_acquire(gtc_space* space, const gtc_model_config* cfg, gtc_run** out) {
  if (!out) return fail(GTC_ERR_INVALID, "out is null");
  *out = nullptr;
  if (!space || !cfg) return fail(GTC_ERR_INVALID, "space/config is null");
  gtc_run* r = nullptr;
  {
    std::lock_guard<std::mutex> lk(space->pool_mu);
    for (size_t i = space->pool.size(); i-- > 0;)
      if (space->pool[i]->cfg.n_max == cfg->n_max) {
        r = space->pool[i];
        space->pool.erase(space->pool.begin() + (std::ptrdiff_t)i);
        break;
      }
  }
  if (!r) return gtc_run_create(space, cfg, out);
  const int rc = gtc_run_reset(r, cfg);
  if (rc) {
    gtc_run_destroy(r);
    return rc;
  }
  *out = r;
  return GTC_OK;
}

extern "C" int gtc_run_release(gtc_run* r) {
  if (!r) return GTC_OK;
  cudaSetDevice(r->space->device);
  if (cudaStreamSynchronize(r->stream) != cudaSuccess) {  // not reusable
    cudaGetLastError();
    return gtc_run_destroy(r);
  }
  std::lock_guard<std::mutex> lk(r->space->pool_mu);
  r->space->pool.push_back(r);
  return GTC_OK;
}

extern "C" int gtc_run_reset(gtc_run* r, const gtc_model_config* cfg) {
  if (!r || !cfg) return fail(GTC_ERR_INVALID, "run/config is null");
  if (cfg->n_max != r->cfg.n_max) return fail(GTC_ERR_CONFIG, "gtc_run_reset cannot change n_max");
  int rc = check_kernel(&cfg->kernel);
  if (rc) return rc;
  if (!(cfg->noise >= 0.0)) return fail(GTC_ERR_INVALID, "GP fit: noise must be non-negative");
  if (!(cfg->jitter > 0.0)) return fail(GTC_ERR_INVALID, "GP fit: jitter must be positive");
  GTC_CUDA(cudaSetDevice(r->space->device));
  const int64_t words = (r->space->n + 31) / 32;
  GTC_CUDA(cudaMemsetAsync(r->visited, 0, words * sizeof(uint32_t), r->stream));
  GTC_CUDA(cudaMemsetAsync(r->acc, 0, 2 * sizeof(VarAccum), r->stream));
  GTC_CUDA(cudaStreamSynchronize(r->stream));
  r->cfg = *cfg;
  r->jitter = cfg->jitter;
  r->n = 0;
  r->predictions_valid = false;
  r->stats_stale = -1;
  r->acc_gen = 0;
  r->acc_valid = false;
  r->visited_host.assign(words, 0u);
  r->visited_count = 0;
  r->first_hint = 0;
  r->ex_host.clear();
  r->y_host.clear();
  r->x_host.clear();
  r->shard_offset = 0;
  r->comm = nullptr;
  r->n_global = 0;
  r->group = nullptr;
  r->has_values = false;
  r->port = PortDev{};
  r->pdl = true;
  r->pass_timed = r->step_timed = r->step_appended = false;
  return GTC_OK;
}

// Host copy of the training set: explicit coordinates (so a shard can hold
// observations of candidates that live on other shards) + raw values.
static void keep_obs(gtc_run* r, int n) {
  r->y_host.resize(n);
  r->x_host.resize((size_t)n * r->space->d);
}
static void push_obs(gtc_run* r, const double* x, double y) {
  r->y_host.push_back(y);
  r->x_host.insert(r->x_host.end(), x, x + r->space->d);
}

static int upload_train(gtc_run* r) {
  const int n = (int)r->y_host.size();
  if (n > 0) {
    GTC_CUDA(cudaMemcpyAsync(r->gp.dev.train_x, r->x_host.data(), r->x_host.size() * sizeof(double),
                             cudaMemcpyHostToDevice, r->stream));
    GTC_CUDA(cudaMemcpyAsync(r->gp.dev.y, r->y_host.data(), sizeof(double) * n, cudaMemcpyHostToDevice, r->stream));
    GTC_CUDA(cudaStreamSynchronize(r->stream));
  }
  return GTC_OK;
}

// Full refit of the run's observations (GpModel::fit semantics) starting at
// `start_jitter`, then the full predictive pass.
static int refit(gtc_run* r, double start_jitter, gtc_fit_info* info) {
  const int n = (int)r->y_host.size();
  r->stats_stale = -1;  // (the factorisation recomputes them)
  int rc = upload_train(r);
  if (rc) return rc;
  // the kernel values need only the training coordinates (and no jitter):
  // they run on the side stream while the single-CTA factorisation (and its
  // escalation round trips) run on the run's stream
  // (launched after the factor kernel: its one large CTA gets an SM before
  // the kernel values' grid fills them)
  const bool kstar = r->side && rebuild_wide_taken(r->space->dev(), n);
  bool forked = false;
  if (kstar) GTC_CUDA(cudaEventRecord(r->ev_fork, r->stream));
  rc = factor_with_escalation(r->gp, r->cfg.kernel, r->cfg.noise, r->cfg.jitter, start_jitter, n, r->stream,
                              [&]() -> int {
                                if (!kstar) return GTC_OK;
                                GTC_CUDA(cudaStreamWaitEvent(r->side, r->ev_fork, 0));
                                launch_kstar(r->space->dev(), r->gp.dev, kparams(r->cfg.kernel), r->V,
                                             r->tile_stride, n, r->side);
                                GTC_LAUNCHED();
                                GTC_CUDA(cudaEventRecord(r->ev_join, r->side));
                                forked = true;
                                return GTC_OK;
                              });
  if (forked) GTC_CUDA(cudaStreamWaitEvent(r->stream, r->ev_join, 0));  // (also on failure: V is the run's again)
  if (rc) {
    r->predictions_valid = false;
    return rc;
  }
  r->n = n;
  r->jitter = r->gp.h_sc->jitter;
  const VarPartials vp = r->vp();
  rc = rebuild_predictions(r->space->dev(), r->gp, r->cfg.kernel, r->V, r->tile_stride, n, r->mu, r->var, &vp,
                           r->tstat, r->stream, forked);
  if (rc) return rc;
  r->predictions_valid = true;
  r->acc_valid = true;
  fill_info(info, *r->gp.h_sc, n, 1);
  return GTC_OK;
}

extern "C" int gtc_fit(gtc_run* r, const int64_t* positions, const double* y_raw, int32_t n,
                       gtc_fit_info* info) {
  if (!r) return fail(GTC_ERR_INVALID, "run is null");
  if (n > r->cfg.n_max) return fail(GTC_ERR_CAPACITY, "more observations than the run's n_max");
  int rc = check_fit_inputs(y_raw, n, r->cfg.noise, r->cfg.jitter);
  if (rc) return rc;
  GTC_CUDA(cudaSetDevice(r->space->device));
  r->stats_stale = -1;  // (a fit replaces the model; n == 0 sets the prior scalars below)
  keep_obs(r, 0);
  for (int i = 0; i < n; ++i) {
    if (positions[i] < 0 || positions[i] >= r->space->n)
      return fail(GTC_ERR_INVALID, "training position out of range");
    push_obs(r, &r->space->host_coords[(size_t)positions[i] * r->space->d], y_raw[i]);
  }
  if (n == 0) {
    r->n = 0;
    r->jitter = r->cfg.jitter;
    std::memset(r->gp.h_sc, 0, sizeof(GpScalars));
    r->gp.h_sc->y_std = 1.0;
    r->gp.h_sc->jitter = r->jitter;
    GTC_CUDA(cudaMemcpyAsync(r->gp.dev.sc, r->gp.h_sc, sizeof(GpScalars), cudaMemcpyHostToDevice, r->stream));
    rc = rebuild_predictions(r->space->dev(), r->gp, r->cfg.kernel, r->V, r->tile_stride, 0, r->mu, r->var, nullptr, r->tstat,
                             r->stream);
    if (rc) return rc;
    GTC_CUDA(cudaStreamSynchronize(r->stream));
    r->predictions_valid = true;
    r->acc_valid = false;
    fill_info(info, *r->gp.h_sc, 0, 1);
    return GTC_OK;
  }
  return refit(r, r->cfg.jitter, info);
}

// CUDA events between the observe path's kernels (gtc_last_pass_ms /
// gtc_last_step_ms / gtc_last_phase_ms) only with GTC_PHASE_EVENTS=1: an
// event between two kernels stops the second from launching early (PDL).
static bool phase_events() {
  static const bool on = [] {
    const char* e = std::getenv("GTC_PHASE_EVENTS");
    return e && e[0] == '1';
  }();
  return on;
}

// Enqueues the bordered-row update + predictive pass for observation n0
// (asynchronous; the pass is a no-op if the pivot fails on the device).
static int enqueue_append(gtc_run* r, int64_t pos, double y_raw, uint32_t* mark) {
  const int n0 = r->n;
  r->stats_stale = -1;  // (the bordered row recomputes the standardisation and beta of rows [0, n0])
  launch_gp_append(r->gp.dev, kparams(r->cfg.kernel), r->cfg.noise, r->space->dev(), pos, nullptr, y_raw, n0,
                   mark, r->stream, r->V, r->tile_stride);
  GTC_LAUNCHED();
  const bool ev = phase_events();
  if (ev) GTC_CUDA(cudaEventRecord(r->ev0, r->stream));
  const VarPartials vp = r->vp();
  launch_extend(r->space->dev(), r->gp.dev, kparams(r->cfg.kernel), r->V, r->tile_stride, n0, 1, true, r->mu,
                r->var, true, &vp, r->tstat, r->stream);
  GTC_LAUNCHED();
  if (ev) GTC_CUDA(cudaEventRecord(r->ev1, r->stream));
  r->pass_timed = ev;
  r->acc_valid = true;  // (stale if the pivot failed; the refit rewrites them)
  return GTC_OK;
}

extern "C" int gtc_append(gtc_run* r, int64_t pos, double y_raw, gtc_fit_info* info) {
  if (!r) return fail(GTC_ERR_INVALID, "run is null");
  if (pos < 0 || pos >= r->space->n) return fail(GTC_ERR_INVALID, "position out of range");
  if (!std::isfinite(y_raw)) return fail(GTC_ERR_INVALID, "GP fit: observations must be finite");
  if (r->n >= r->cfg.n_max) return fail(GTC_ERR_CAPACITY, "more observations than the run's n_max");
  GTC_CUDA(cudaSetDevice(r->space->device));
  const int n0 = r->n;
  keep_obs(r, n0);
  push_obs(r, &r->space->host_coords[(size_t)pos * r->space->d], y_raw);
  if (n0 == 0) return refit(r, r->cfg.jitter, info);
  int rc = enqueue_append(r, pos, y_raw, nullptr);
  if (rc) return rc;
  GTC_CUDA(cudaMemcpyAsync(r->gp.h_sc, r->gp.dev.sc, sizeof(GpScalars), cudaMemcpyDeviceToHost, r->stream));
  GTC_CUDA(cudaStreamSynchronize(r->stream));
  if (r->gp.h_sc->status != 0) {
    // new pivot <= 0 at the current jitter: the reference's refit would fail at
    // every jitter up to the current one too, so escalate from jitter * 2.
    return refit(r, r->jitter * 2.0, info);
  }
  r->n = n0 + 1;
  r->predictions_valid = true;
  fill_info(info, *r->gp.h_sc, r->n, 0);
  return GTC_OK;
}

static int flush_stats(gtc_run* r);

extern "C" int gtc_truncate(gtc_run* r, int32_t n, gtc_fit_info* info) {
  if (!r) return fail(GTC_ERR_INVALID, "run is null");
  if (n < 0 || n > r->n) return fail(GTC_ERR_INVALID, "truncate: n out of range");
  GTC_CUDA(cudaSetDevice(r->space->device));
  if (n == 0) return gtc_fit(r, nullptr, nullptr, 0, info);
  if (r->jitter != r->cfg.jitter) {
    // the factor was escalated past the base jitter by a later observation:
    // GpModel::fit of the prefix restarts at the base jitter (gp.hpp:116-129)
    keep_obs(r, n);
    return refit(r, r->cfg.jitter, info);
  }
  r->n = n;
  keep_obs(r, n);
  r->predictions_valid = false;
  r->stats_stale = n;  // (a following append recomputes them: nothing to launch now)
  if (info) {  // the scalars need a round trip; without `info` the call stays asynchronous
    if (int rc = flush_stats(r)) return rc;
    GTC_CUDA(cudaMemcpyAsync(r->gp.h_sc, r->gp.dev.sc, sizeof(GpScalars), cudaMemcpyDeviceToHost, r->stream));
    GTC_CUDA(cudaStreamSynchronize(r->stream));
    fill_info(info, *r->gp.h_sc, n, 0);
  }
  return GTC_OK;
}

static int flush_stats(gtc_run* r) {
  if (r->stats_stale < 0) return GTC_OK;
  launch_gp_truncate(r->gp.dev, r->stats_stale, r->stream);
  GTC_LAUNCHED();
  r->stats_stale = -1;
  return GTC_OK;
}

static int ensure_predictions(gtc_run* r) {
  if (int rc = flush_stats(r)) return rc;
  if (r->predictions_valid) return GTC_OK;
  if (r->n == 0) {
    launch_prior(r->mu, r->var, r->space->n_pad, r->cfg.kernel.output_variance, r->tstat, r->stream);
    r->acc_valid = false;
  } else {
    // posterior from the resident V rows (r = 0 new rows)
    const VarPartials vp = r->vp();
    launch_extend(r->space->dev(), r->gp.dev, kparams(r->cfg.kernel), r->V, r->tile_stride, r->n, 0, true,
                  r->mu, r->var, false, &vp, r->tstat, r->stream);
    r->acc_valid = true;
  }
  GTC_LAUNCHED();
  r->predictions_valid = true;
  return GTC_OK;
}

static bool host_mark(gtc_run* r, int64_t pos, int set) {
  uint32_t& w = r->visited_host[pos >> 5];
  const uint32_t bit = 1u << (pos & 31);
  const bool was = (w & bit) != 0;
  if (set && !was) {
    w |= bit;
    ++r->visited_count;
    return true;
  }
  if (!set && was) {
    w &= ~bit;
    --r->visited_count;
    r->first_hint = std::min(r->first_hint, pos);
    return true;
  }
  return false;
}

static int set_visited(gtc_run* r, int64_t pos, int set) {
  if (!r) return fail(GTC_ERR_INVALID, "run is null");
  if (pos < 0 || pos >= r->space->n) return fail(GTC_ERR_INVALID, "position out of range");
  GTC_CUDA(cudaSetDevice(r->space->device));
  if (!host_mark(r, pos, set)) return GTC_OK;
  VarAccum* acc = r->live_acc();
  launch_mark(r->visited, pos, set, r->stream, acc, r->var, r->cfg.kernel.output_variance);
  GTC_LAUNCHED();
  r->acc_valid = acc != nullptr;
  return GTC_OK;
}

extern "C" int gtc_mark_visited(gtc_run* r, int64_t pos) { return set_visited(r, pos, 1); }
extern "C" int gtc_unmark_visited(gtc_run* r, int64_t pos) { return set_visited(r, pos, 0); }
extern "C" int64_t gtc_unvisited_count(const gtc_run* r) {
  return r ? r->space->n - r->visited_count : -1;
}

extern "C" int gtc_mean_variance(gtc_run* r, double* out, int64_t* count) {
  if (!r || !out) return fail(GTC_ERR_INVALID, "null argument");
  GTC_CUDA(cudaSetDevice(r->space->device));
  int rc = ensure_predictions(r);
  if (rc) return rc;
  launch_varsum(r->var, r->visited, r->space->n, r->red.vsum, r->red.vcnt, r->red.vcounter, r->red.totals, r->stream);
  GTC_LAUNCHED();
  GTC_CUDA(cudaMemcpyAsync(r->red.h_totals, r->red.totals, sizeof(VarTotals), cudaMemcpyDeviceToHost, r->stream));
  GTC_CUDA(cudaStreamSynchronize(r->stream));
  // strategies.hpp:394-397: empty candidate set -> 0.0
  *out = r->red.h_totals->count > 0 ? r->red.h_totals->sum / (double)r->red.h_totals->count : 0.0;
  if (count) *count = r->red.h_totals->count;
  return GTC_OK;
}

// First unvisited position >= p (n if none), from the host's visited bitmap.
static int64_t first_unvisited_from(const gtc_run* r, int64_t p) {
  const int64_t n = r->space->n;
  while (p < n) {
    const uint32_t w = r->visited_host[p >> 5] | ((1u << (p & 31)) - 1u);  // bits below p: skip
    if (w != 0xffffffffu) return std::min<int64_t>(n, (p & ~int64_t(31)) + __builtin_ctz(~w));
    p = (p | 31) + 1;
  }
  return n;
}

// The first eligible position (portfolio.hpp:52's first candidate; -1 if
// none) and the eligible count, from the host's visited bookkeeping and the
// sorted exclusion list: the device selection does not have to reduce them.
static void first_and_count(gtc_run* r, const std::vector<int64_t>& ex, int64_t* first, int64_t* count) {
  const int64_t n = r->space->n;
  auto visited = [&](int64_t q) { return (r->visited_host[q >> 5] >> (q & 31)) & 1u; };
  int64_t ex_unvisited = 0;
  for (int64_t e : ex) ex_unvisited += visited(e) ? 0 : 1;
  *count = n - r->visited_count - ex_unvisited;
  r->first_hint = first_unvisited_from(r, r->first_hint);
  int64_t q = r->first_hint;
  while (q < n && std::binary_search(ex.begin(), ex.end(), q)) q = first_unvisited_from(r, q + 1);
  *first = q < n ? q : -1;
}

// Makes the run's current variance total match its visited set.
static int ensure_var_totals(gtc_run* r) {
  if (r->acc_valid) return GTC_OK;  // visited set unchanged since the last pass
  launch_var_partials(r->var, r->space->n, r->cfg.kernel.output_variance, r->vp(), r->stream);
  GTC_LAUNCHED();
  r->acc_valid = true;
  return GTC_OK;
}

static int build_selection(gtc_run* r, const gtc_select_args* a, bool global_totals, double global_sum,
                           long long global_count, SelectRunArgs* out) {
  int rc = ensure_predictions(r);
  if (rc) return rc;
  SelectParams p{a->af_mask & 7u, a->lambda_mode, a->lambda_constant, a->cv_initial_sample_mean,
                 a->cv_initial_mean_variance, a->f_best_raw, nullptr, 0, -1, 0};
  // exclusions: sorted, unique, in range (the device tests membership)
  std::vector<int64_t>& ex = r->ex_host;
  ex.clear();
  for (int32_t k = 0; k < a->n_excluded; ++k)
    if (a->excluded[k] >= 0 && a->excluded[k] < r->space->n) ex.push_back(a->excluded[k]);
  std::sort(ex.begin(), ex.end());
  ex.erase(std::unique(ex.begin(), ex.end()), ex.end());
  if (!ex.empty()) {
    if ((int)ex.size() > r->excluded_cap) {
      cudaFree(r->excluded);
      r->excluded = nullptr;
      r->excluded_cap = 0;
      if ((rc = dalloc(&r->excluded, ex.size()))) return rc;
      r->excluded_cap = (int)ex.size();
    }
    GTC_CUDA(cudaMemcpyAsync(r->excluded, ex.data(), sizeof(int64_t) * ex.size(), cudaMemcpyHostToDevice, r->stream));
    p.excluded = r->excluded;
    p.n_excluded = (int)ex.size();
  }
  first_and_count(r, ex, &p.first_eligible, &p.n_candidates);
  VarSource vs{nullptr, 0.0, global_sum, global_count, 1};
  if (!global_totals) {
    if ((rc = ensure_var_totals(r))) return rc;
    vs = r->vsrc();
  }
  *out = SelectRunArgs{r->mu, r->var, r->visited, r->space->n, r->gp.dev.sc, p, vs, r->tstat, r->red.b, r->red.sel};
  return GTC_OK;
}

// Enqueues the selection kernel (asynchronous).  With `global_totals`, the
// mean variance comes from the global (sum, count) passed by value
// (candidate-axis sharding) instead of this run's own variance total.
static int enqueue_selection(gtc_run* r, const gtc_select_args* a, bool global_totals = false,
                             double global_sum = 0.0, long long global_count = 0, uint32_t host_seq = 0) {
  SelectRunArgs sa;
  int rc = build_selection(r, a, global_totals, global_sum, global_count, &sa);
  if (rc) return rc;
  if (host_seq) {  // the last block writes the record + scalars into h_rb, then the sequence word
    sa.p.host_sel = &r->h_rb->sel;
    sa.p.host_sc = &r->h_rb->sc;
    sa.p.host_seq = &r->h_rb->seq;
    sa.p.seq = host_seq;
  }
  launch_select(sa.mu, sa.var, sa.visited, sa.n, sa.sc, sa.p, sa.vs, sa.tstat, sa.b, sa.out, r->stream);
  GTC_LAUNCHED();
  return GTC_OK;
}

// =============================================================== resident loop

extern "C" int gtc_run_set_pdl(gtc_run* r, int32_t enable) {
  if (!r) return fail(GTC_ERR_INVALID, "run is null");
  r->pdl = enable != 0;
  return GTC_OK;
}

extern "C" int gtc_run_set_portfolio(gtc_run* r, const gtc_portfolio_config* c) {
  if (!r) return fail(GTC_ERR_INVALID, "run is null");
  r->port = PortDev{};
  if (!c || c->mode == GTC_PORTFOLIO_NONE) return GTC_OK;
  if (c->mode != GTC_PORTFOLIO_MULTI && c->mode != GTC_PORTFOLIO_ADVANCED)
    return fail(GTC_ERR_CONFIG, "unknown portfolio mode");
  // PortfolioConfig checks (portfolio.hpp:101-110)
  if (c->skip_threshold < 1) return fail(GTC_ERR_CONFIG, "skip threshold must be >= 1");
  if (!(c->discount > 0.0 && c->discount < 1.0)) return fail(GTC_ERR_CONFIG, "discount factor must be in (0,1)");
  if (!(c->required_improvement > 0.0)) return fail(GTC_ERR_CONFIG, "required improvement factor must be positive");
  r->port.mode = c->mode;
  r->port.skip_threshold = c->skip_threshold;
  r->port.discount = c->discount;
  r->port.rho = c->required_improvement;
  for (int a = 0; a < 3; ++a) {
    r->port.active[a] = 1;
    r->port.last_sug[a] = -1;
  }
  return GTC_OK;
}

extern "C" int gtc_portfolio_trace(int device, const gtc_portfolio_config* c, const int32_t* initial_active,
                                   int32_t n_ops, const gtc_portfolio_op* ops, gtc_portfolio_state* out) {
  static_assert(sizeof(PortOp) == sizeof(gtc_portfolio_op), "op layout");
  static_assert(sizeof(PortState) == sizeof(gtc_portfolio_state), "state layout");
  if (!c || (n_ops > 0 && (!ops || !out)) || n_ops < 0) return fail(GTC_ERR_INVALID, "null argument");
  if (c->mode != GTC_PORTFOLIO_MULTI && c->mode != GTC_PORTFOLIO_ADVANCED)
    return fail(GTC_ERR_CONFIG, "unknown portfolio mode");
  if (c->skip_threshold < 1) return fail(GTC_ERR_CONFIG, "skip threshold must be >= 1");
  if (!(c->discount > 0.0 && c->discount < 1.0)) return fail(GTC_ERR_CONFIG, "discount factor must be in (0,1)");
  if (!(c->required_improvement > 0.0)) return fail(GTC_ERR_CONFIG, "required improvement factor must be positive");
  for (int32_t i = 0; i < n_ops; ++i)
    if (ops[i].kind == 1 && (ops[i].af < 0 || ops[i].af > 2)) return fail(GTC_ERR_INVALID, "unknown acquisition function");
  if (n_ops == 0) return GTC_OK;
  GTC_CUDA(cudaSetDevice(device));
  PortDev P{};
  P.mode = c->mode;
  P.skip_threshold = c->skip_threshold;
  P.discount = c->discount;
  P.rho = c->required_improvement;
  for (int a = 0; a < 3; ++a) {
    P.active[a] = initial_active ? (initial_active[a] != 0) : 1;
    P.last_sug[a] = -1;
  }
  PortOp* d_ops = nullptr;
  PortState* d_out = nullptr;
  int rc;
  if ((rc = dalloc(&d_ops, (size_t)n_ops)) || (rc = dalloc(&d_out, (size_t)n_ops))) {
    cudaFree(d_ops);
    return rc;
  }
  cudaError_t e = cudaMemcpy(d_ops, ops, sizeof(PortOp) * (size_t)n_ops, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    launch_portfolio_trace(P, d_ops, n_ops, d_out, nullptr);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, d_out, sizeof(PortState) * (size_t)n_ops, cudaMemcpyDeviceToHost);
  cudaFree(d_ops);
  cudaFree(d_out);
  if (e != cudaSuccess) return fail(GTC_ERR_CUDA, std::string("portfolio trace: ") + cudaGetErrorString(e));
  return GTC_OK;
}

extern "C" int gtc_run_set_values(gtc_run* r, const double* values, int64_t n) {
  if (!r || !values) return fail(GTC_ERR_INVALID, "null argument");
  const int64_t want = r->comm ? r->n_global : r->space->n;  // sharded: the GLOBAL table
  if (n != want) return fail(GTC_ERR_INVALID, "value table size != space size");
  GTC_CUDA(cudaSetDevice(r->space->device));
  int rc;
  if (r->d_values && r->values_cap < n) {
    cudaFree(r->d_values);
    r->d_values = nullptr;
  }
  if (!r->d_values && (rc = dalloc(&r->d_values, (size_t)n))) return rc;
  r->values_cap = n;
  GTC_CUDA(cudaMemcpyAsync(r->d_values, values, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, r->stream));
  GTC_CUDA(cudaStreamSynchronize(r->stream));
  r->has_values = true;
  return GTC_OK;
}

// Host bookkeeping of the steps a resident chunk ran (the same updates
// gtc_observe makes per call).
// Sharded runs: positions are global, the marks land on the owning shard
// only and the coordinates come from the step's record (xrec).
static void replay_steps(gtc_run* r, const StepRec* rec, int m, bool hold, int hold_n0, int64_t* hold_prev,
                         const double* xrec = nullptr) {
  const int64_t off = r->comm ? r->shard_offset : 0;
  auto local = [&](int64_t pos) -> int64_t {
    const int64_t p = pos - off;
    return p >= 0 && p < r->space->n ? p : -1;
  };
  for (int i = 0; i < m; ++i) {
    const int64_t pos = rec[i].position;
    const int64_t lp = local(pos);
    if (rec[i].valid) {
      if (hold) {
        if (*hold_prev >= 0 && local(*hold_prev) >= 0) host_mark(r, local(*hold_prev), 0);
        *hold_prev = pos;
        keep_obs(r, hold_n0);
      }
      push_obs(r, xrec ? xrec + (size_t)i * r->space->d : &r->space->host_coords[(size_t)pos * r->space->d],
               rec[i].value);
    }
    if (lp >= 0) host_mark(r, lp, 1);
  }
}

// k BO iterations of a single-AF strategy in simulation mode without host
// round trips: per step select (its last block advances the loop state:
// table lookup, visited mark, f_best) -> bordered append -> predictive pass,
// all launch arguments constant, chained by programmatic dependent launch.  A failed bordered pivot halts the chunk on the device; the host
// refactorises with escalated jitter (gp.hpp:116-129, as gtc_append) and
// continues with a new chunk.
extern "C" int gtc_run_steps(gtc_run* r, const gtc_select_args* a, int32_t k, int32_t flags,
                             gtc_step_record* records, int32_t* done, gtc_fit_info* info) {
  if (!r || !a || !done || (k > 0 && !records)) return fail(GTC_ERR_INVALID, "null argument");
  *done = 0;
  const bool portfolio = r->port.mode != 0;
  // a portfolio consults every function's argmax: the selection computes all three
  const uint32_t mask = portfolio ? 7u : a->af_mask & 7u;
  if (!portfolio && (mask == 0 || (mask & (mask - 1)) != 0))
    return fail(GTC_ERR_INVALID, "gtc_run_steps needs exactly one acquisition function (or a portfolio)");
  if (portfolio && (flags & GTC_STEPS_HOLD_N)) return fail(GTC_ERR_INVALID, "hold mode is single-AF only");
  if (a->n_excluded > 0) return fail(GTC_ERR_INVALID, "gtc_run_steps takes no exclusions");
  if (!r->has_values) return fail(GTC_ERR_INVALID, "no value table (gtc_run_set_values)");
  if (r->n < 1) return fail(GTC_ERR_INVALID, "gtc_run_steps needs a fitted model (n >= 1)");
  const bool hold = (flags & GTC_STEPS_HOLD_N) != 0;
  if (hold && r->n >= r->cfg.n_max) return fail(GTC_ERR_CAPACITY, "more observations than the run's n_max");
  if (k <= 0) return GTC_OK;
  GTC_CUDA(cudaSetDevice(r->space->device));
  set_thread_pdl(r->pdl);
  int rc;
  if (k > r->rec_cap) {  // (cudaFree synchronises the device: grow rarely)
    const int cap = std::max({k, r->cfg.n_max, 2 * r->rec_cap});
    cudaFree(r->d_rec);
    r->d_rec = nullptr;
    r->rec_cap = 0;
    if ((rc = dalloc(&r->d_rec, (size_t)cap))) return rc;
    r->rec_cap = cap;
  }
  if (!r->d_loop) {
    if ((rc = dalloc(&r->d_loop, 1))) return rc;
    GTC_CUDA(cudaMallocHost(&r->h_loop, sizeof(LoopDev)));
  }
  if (portfolio && !r->d_sorted_y && (rc = dalloc(&r->d_sorted_y, (size_t)r->cfg.n_max))) return rc;
  const bool sharded = r->comm != nullptr;
  const int d = r->space->d;
  if (sharded && r->xrec_cap < k) {
    cudaFree(r->d_xrec);
    r->d_xrec = nullptr;
    r->xrec_cap = 0;
    if ((rc = dalloc(&r->d_xrec, (size_t)k * d))) return rc;
    r->xrec_cap = k;
  }
  const int64_t rec_bytes = shard_record_bytes(mask, d, r->cfg.n_max);
  int af = 0;
  while (!((mask >> af) & 1u)) ++af;
  const int hold_n0 = r->n;  // hold: every valid step appends at this row
  int64_t hold_prev = -1;
  double f_best = a->f_best_raw;
  bool refitted = false;
  while (*done < k) {
    const int m = k - *done;
    if (!sharded && r->space->n - r->visited_count <= 0) break;  // (sharded: the merge halts on the global count)
    if ((rc = ensure_predictions(r)) || (rc = ensure_var_totals(r))) return rc;
    const bool timing = (flags & GTC_STEPS_TIMING) != 0;
    // graph-launched chunks (see below) size for the largest row, so that one
    // captured graph serves every chunk of the run handle
    bool graphed = !r->pdl && !timing && !r->graphs.failed && !sharded;
    const int n0_max = hold ? hold_n0 : graphed ? r->cfg.n_max - 1 : std::min(r->n + m - 1, r->cfg.n_max - 1);
    LoopDev& L = *r->h_loop;
    L = LoopDev{};
    L.pos = -1;
    L.n = r->n;
    L.gen = r->acc_gen;
    L.halt = kLoopRunning;
    L.af = af;
    L.n_max = r->cfg.n_max;
    L.hold = hold ? 1 : 0;
    L.hold_n0 = hold_n0;
    L.hold_prev = hold_prev;
    L.f_best = f_best;
    L.f_base = a->f_best_raw;
    r->first_hint = first_unvisited_from(r, r->first_hint);
    L.first = r->first_hint < r->space->n ? r->first_hint : -1;
    L.count = r->space->n - r->visited_count;
    L.n_space = r->space->n;
    L.acc = r->acc;
    L.table = r->d_values;
    L.visited = r->visited;
    L.var = r->var;
    L.s2 = r->cfg.kernel.output_variance;
    L.sc = r->gp.dev.sc;
    L.sel = r->red.sel;
    L.rec = r->d_rec;
    L.port = r->port;
    if (portfolio) {  // the valid observations = the model's training values, sorted (median)
      std::vector<double>& ys = r->sorted_host;
      ys.assign(r->y_host.begin(), r->y_host.end());
      std::sort(ys.begin(), ys.end());
      GTC_CUDA(cudaMemcpyAsync(r->d_sorted_y, ys.data(), sizeof(double) * ys.size(), cudaMemcpyHostToDevice,
                               r->stream));
      L.sorted_y = r->d_sorted_y;
      L.n_sorted = (int32_t)ys.size();
    }
    L.lambda_mode = a->lambda_mode;
    L.lambda_constant = a->lambda_constant;
    L.cv_mu_s = a->cv_initial_sample_mean;
    L.cv_var_s = a->cv_initial_mean_variance;
    L.g = r->gp.dev;  // the selection's last block appends valid steps from the pick's V column
    L.kp = kparams(r->cfg.kernel);
    L.noise = r->cfg.noise;
    L.sp = r->space->dev();
    L.V = r->V;
    L.tile_stride = r->tile_stride;
    if (sharded) {
      L.nranks = r->comm->nranks;
      L.offset = r->shard_offset;
      L.send = r->d_send;
      L.recv = r->d_recv;
      L.rec_bytes = rec_bytes;
      L.gacc = r->d_gacc;
      L.xrec = r->d_xrec;
      L.gsel = r->red.sel;
    }
    L.sel_mask = mask;
    // one device: the selection's last block appends valid picks (no append
    // kernel per step); sharded: the merge kernel + the append kernel do
    L.fused_append = sharded ? 0 : 1;
    const int fused_n_max = sharded ? 0 : r->cfg.n_max;
    GTC_CUDA(cudaMemcpyAsync(r->d_loop, r->h_loop, sizeof(LoopDev), cudaMemcpyHostToDevice, r->stream));
    // (every per-run / per-step selection input is read from the loop state:
    // the launch arguments depend only on the run handle and its model config)
    SelectParams p{mask, 0, 0.0, 0.0, 0.0, 0.0, nullptr, 0, -1, 0, r->d_loop};
    if (!sharded) {  // L2 warm-up of the winners' table entries and V columns (rows < n0_max)
      p.pf_table = r->d_values;
      p.pf_V = r->V;
      p.pf_tile_stride = r->tile_stride;
      p.pf_rows = n0_max;
      p.pf_gp[0] = r->gp.dev.c;
      p.pf_gp[1] = r->gp.dev.e;
      p.pf_gp[2] = r->gp.dev.y;
    }
    VarSource vs = r->vsrc();
    vs.acc = r->acc;  // loop mode: both generations (the kernel picks the loop state's)
    // loop-mode launch arguments: per-step values come from the loop state
    // (the bordered append runs in the selection's last block, or in the
    // sharded merge kernel)
    ExtendArgs ea = make_pass_args(r->space->dev(), r->gp.dev, kparams(r->cfg.kernel), r->V, r->tile_stride, n0_max,
                                   r->mu, r->var, nullptr, r->tstat);
    ea.visited = r->visited;
    ea.acc = r->acc;  // (generation chosen on the device)
    ea.acc_clear = r->acc + 1;
    ea.loop = r->d_loop;
    if (timing) {
      while ((int)r->step_events.size() < 3 * m + 1) {
        cudaEvent_t ev;
        GTC_CUDA(cudaEventCreate(&ev));
        r->step_events.push_back(ev);
      }
      r->timed_steps = 0;
    }
    cudaEvent_t* te = r->step_events.data();
    auto launch_iteration = [&]() -> int {
      launch_select(r->mu, r->var, r->visited, r->space->n, r->gp.dev.sc, p, vs, r->tstat, r->red.b, r->red.sel,
                    r->stream, fused_n_max);
      launch_extend_loop(ea, r->space->n_pad / kTile, r->cfg.kernel.nu, r->stream);
      GTC_LAUNCHED();
      return GTC_OK;
    };
    // Runs driven by many host threads (no PDL) are bound by the driver's
    // launch rate: launch captured graphs of kSteps iterations instead
    // (identical kernels and arguments, one launch per kSteps iterations).
    constexpr int kSteps = 16;
    if (graphed) {
      char key[256];
      std::snprintf(key, sizeof key, "%u|%d|%d|%d|%.17g|%.17g|%.17g", mask, n0_max, hold ? 1 : 0,
                    r->cfg.kernel.nu, r->cfg.kernel.lengthscale, r->cfg.kernel.output_variance, r->cfg.noise);
      if (r->graphs.key != key) {
        r->graphs.release();
        auto capture = [&](int count, cudaGraphExec_t* out) -> bool {
          if (cudaStreamBeginCapture(r->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return false;
          int lrc = GTC_OK;
          for (int i = 0; i < count && lrc == GTC_OK; ++i) lrc = launch_iteration();
          cudaGraph_t g = nullptr;
          const bool ok = cudaStreamEndCapture(r->stream, &g) == cudaSuccess && lrc == GTC_OK && g &&
                          cudaGraphInstantiate(out, g, 0) == cudaSuccess;
          if (g) cudaGraphDestroy(g);
          return ok;
        };
        if (capture(kSteps, &r->graphs.many) && capture(1, &r->graphs.one)) {
          r->graphs.key = key;
        } else {  // fall back to plain launches for this run handle
          cudaGetLastError();
          r->graphs.release();
          r->graphs.failed = true;
          graphed = false;
        }
      }
    }
    GTC_CUDA(cudaEventRecord(r->ev_step0, r->stream));
    if (sharded) {
      // per step: local selection -> all-gather of the records -> merge + loop
      // advance + column row -> (exact row fallback) -> local pass -> all-gather
      // of the accumulators; the chunk starts with the accumulators' exchange
      const size_t acc_bytes = 2 * sizeof(VarAccum);
      if ((rc = r->comm->allgather(r->acc, r->d_gacc, acc_bytes, r->stream))) return rc;
      for (int i = 0; i < m; ++i) {
        if (timing) GTC_CUDA(cudaEventRecord(te[3 * i], r->stream));
        launch_select(r->mu, r->var, r->visited, r->space->n, r->gp.dev.sc, p, vs, r->tstat, r->red.b, r->red.sel,
                      r->stream);
        GTC_LAUNCHED();
        if ((rc = r->comm->allgather(r->d_send, r->d_recv, (size_t)rec_bytes, r->stream))) return rc;
        launch_shard_merge(r->d_loop, r->cfg.kernel.nu, r->cfg.n_max, r->stream);  // + the bordered append
        if (timing) {
          GTC_CUDA(cudaEventRecord(te[3 * i + 1], r->stream));
          GTC_CUDA(cudaEventRecord(te[3 * i + 2], r->stream));
        }
        launch_extend_loop(ea, r->space->n_pad / kTile, r->cfg.kernel.nu, r->stream);
        GTC_LAUNCHED();
        if ((rc = r->comm->allgather(r->acc, r->d_gacc, acc_bytes, r->stream))) return rc;
      }
    }
    if (graphed) {
      for (int i = 0; i + kSteps <= m; i += kSteps) GTC_CUDA(cudaGraphLaunch(r->graphs.many, r->stream));
      for (int i = m - m % kSteps; i < m; ++i) GTC_CUDA(cudaGraphLaunch(r->graphs.one, r->stream));
    }
    for (int i = 0; i < m && !graphed && !sharded; ++i) {
      if (timing) GTC_CUDA(cudaEventRecord(te[3 * i], r->stream));
      launch_select(r->mu, r->var, r->visited, r->space->n, r->gp.dev.sc, p, vs, r->tstat, r->red.b, r->red.sel,
                    r->stream, fused_n_max);
      if (timing) {  // (the append runs in the selection's last block: an empty phase)
        GTC_CUDA(cudaEventRecord(te[3 * i + 1], r->stream));
        GTC_CUDA(cudaEventRecord(te[3 * i + 2], r->stream));
      }
      launch_extend_loop(ea, r->space->n_pad / kTile, r->cfg.kernel.nu, r->stream);
      GTC_LAUNCHED();
    }
    if (timing) {
      GTC_CUDA(cudaEventRecord(te[3 * m], r->stream));
      r->timed_steps = m;
    }
    GTC_CUDA(cudaEventRecord(r->ev_step1, r->stream));
    r->step_timed = true;
    r->step_appended = false;
    r->pass_timed = false;
    GTC_CUDA(cudaMemcpyAsync(r->h_loop, r->d_loop, sizeof(LoopDev), cudaMemcpyDeviceToHost, r->stream));
    GTC_CUDA(cudaMemcpyAsync(&r->h_rb->sc, r->gp.dev.sc, sizeof(GpScalars), cudaMemcpyDeviceToHost, r->stream));
    static_assert(sizeof(StepRec) == sizeof(gtc_step_record), "record layout");
    GTC_CUDA(cudaMemcpyAsync(records + *done, r->d_rec, sizeof(StepRec) * (size_t)m, cudaMemcpyDeviceToHost, r->stream));
    if (sharded) {
      r->xrec_host.resize((size_t)m * d);
      GTC_CUDA(cudaMemcpyAsync(r->xrec_host.data(), r->d_xrec, sizeof(double) * (size_t)m * d, cudaMemcpyDeviceToHost,
                               r->stream));
    }
    GTC_CUDA(cudaStreamSynchronize(r->stream));
    const int steps = L.step;
    replay_steps(r, reinterpret_cast<const StepRec*>(records + *done), steps, hold, hold_n0, &hold_prev,
                 sharded ? r->xrec_host.data() : nullptr);
    *done += steps;
    r->acc_gen = L.gen;
    r->port = L.port;
    f_best = L.f_best;
    if (L.halt == kLoopPivot) {
      // the last step's bordered row failed (its observation is in the host
      // training set): refactorise from 2 x jitter like gtc_append
      if ((rc = refit(r, r->jitter * 2.0, info))) return rc;
      refitted = true;
      if (hold) return fail(GTC_ERR_CONDITIONING, "gtc_run_steps: bordered pivot failed in hold mode");
      continue;
    }
    r->n = hold ? (hold_prev >= 0 ? hold_n0 + 1 : hold_n0) : L.n;
    if (steps > 0) *r->gp.h_sc = r->h_rb->sc;
    r->predictions_valid = true;
    r->acc_valid = true;
    if (L.halt == kLoopCapacity) return fail(GTC_ERR_CAPACITY, "more observations than the run's n_max");
    if (L.halt == kLoopNoCandidates) break;
  }
  fill_info(info, *r->gp.h_sc, r->n, refitted ? 1 : 0);
  return GTC_OK;
}

extern "C" int gtc_last_steps_phase_ms(const gtc_run* r, double* out3) {
  if (!r || !out3) return fail(GTC_ERR_INVALID, "null argument");
  if (r->timed_steps <= 0) return fail(GTC_ERR_INVALID, "last gtc_run_steps chunk was not timed");
  double acc[3] = {0.0, 0.0, 0.0};
  const cudaEvent_t* te = r->step_events.data();
  for (int i = 0; i < r->timed_steps; ++i)
    for (int k = 0; k < 3; ++k) {
      float ms = 0.f;
      GTC_CUDA(cudaEventElapsedTime(&ms, te[3 * i + k], te[3 * i + k + 1]));
      acc[k] += ms;
    }
  for (int k = 0; k < 3; ++k) out3[k] = acc[k] / r->timed_steps;
  return GTC_OK;
}

extern "C" double gtc_last_steps_ms(const gtc_run* r) {
  if (!r || !r->step_timed) return 0.0;
  float ms = 0.f;
  return cudaEventElapsedTime(&ms, r->ev_step0, r->ev_step1) == cudaSuccess ? (double)ms : 0.0;
}

// =============================================================== sharding

extern "C" int gtc_fit_points(gtc_run* r, const double* X, const double* y_raw, int32_t n, gtc_fit_info* info) {
  if (!r) return fail(GTC_ERR_INVALID, "run is null");
  if (n > r->cfg.n_max) return fail(GTC_ERR_CAPACITY, "more observations than the run's n_max");
  int rc = check_fit_inputs(y_raw, n, r->cfg.noise, r->cfg.jitter);
  if (rc) return rc;
  if (n == 0) return gtc_fit(r, nullptr, nullptr, 0, info);
  GTC_CUDA(cudaSetDevice(r->space->device));
  keep_obs(r, 0);
  for (int i = 0; i < n; ++i) push_obs(r, X + (size_t)i * r->space->d, y_raw[i]);
  return refit(r, r->cfg.jitter, info);
}

extern "C" int gtc_run_set_shard(gtc_run* r, int64_t offset) {
  if (!r || offset < 0) return fail(GTC_ERR_INVALID, "bad shard");
  r->shard_offset = offset;
  return GTC_OK;
}

extern "C" int gtc_run_attach_comm(gtc_run* r, gtc_comm* comm, int64_t offset, int64_t n_global) {
  if (!r) return fail(GTC_ERR_INVALID, "run is null");
  GTC_CUDA(cudaSetDevice(r->space->device));
  GTC_CUDA(cudaStreamSynchronize(r->stream));
  if (!comm) {
    r->comm = nullptr;
    r->n_global = 0;
    r->shard_offset = 0;
    r->has_values = false;
    return GTC_OK;
  }
  if (offset < 0 || offset % kTile != 0)
    return fail(GTC_ERR_INVALID, "shard offset must be a non-negative multiple of 256");
  if (n_global < offset + r->space->n) return fail(GTC_ERR_INVALID, "shard exceeds n_global");
  const int nranks = comm->nranks;
  const int64_t rb = shard_record_bytes(7u, r->space->d, r->cfg.n_max);
  cudaFree(r->d_send);
  cudaFree(r->d_recv);
  cudaFree(r->d_gacc);
  r->d_send = r->d_recv = nullptr;
  r->d_gacc = nullptr;
  int rc;
  if ((rc = dalloc(&r->d_send, (size_t)rb)) || (rc = dalloc(&r->d_recv, (size_t)rb * nranks)) ||
      (rc = dalloc(&r->d_gacc, (size_t)2 * nranks)))
    return rc;
  GTC_CUDA(cudaMemset(r->d_send, 0, (size_t)rb));
  r->comm = comm;
  r->shard_offset = offset;
  r->n_global = n_global;
  r->has_values = false;  // the table must be the global one
  return GTC_OK;
}

// This shard's total of the posterior variance over its unvisited candidates.
static int enqueue_local_totals(gtc_run* r) {
  int rc = ensure_predictions(r);
  if (rc) return rc;
  if ((rc = ensure_var_totals(r))) return rc;
  launch_var_totals(r->vsrc(), r->red.totals, r->stream);
  GTC_LAUNCHED();
  return GTC_OK;
}

extern "C" int gtc_shard_observe(gtc_run* r, const double* x_new, int64_t local_pos, double y_raw, int32_t valid,
                                 double* var_sum, int64_t* var_count, gtc_fit_info* info) {
  if (!r || !x_new || !var_sum || !var_count) return fail(GTC_ERR_INVALID, "null argument");
  if (local_pos >= r->space->n) return fail(GTC_ERR_INVALID, "position out of range");
  if (valid && !std::isfinite(y_raw)) return fail(GTC_ERR_INVALID, "GP fit: observations must be finite");
  if (valid && r->n >= r->cfg.n_max) return fail(GTC_ERR_CAPACITY, "more observations than the run's n_max");
  GTC_CUDA(cudaSetDevice(r->space->device));
  int rc;
  if (local_pos >= 0 && host_mark(r, local_pos, 1)) {
    launch_mark(r->visited, local_pos, 1, r->stream);
    GTC_LAUNCHED();
    r->acc_valid = false;
  }
  const int n0 = r->n;
  bool appended = false;
  if (valid) {
    keep_obs(r, n0);
    push_obs(r, x_new, y_raw);
    if (n0 == 0) {
      if ((rc = refit(r, r->cfg.jitter, info))) return rc;
    } else {
      std::memcpy(r->h_xnew, x_new, sizeof(double) * r->space->d);
      GTC_CUDA(cudaMemcpyAsync(r->d_xnew, r->h_xnew, sizeof(double) * r->space->d, cudaMemcpyHostToDevice, r->stream));
      r->stats_stale = -1;  // (recomputed by the bordered row)
      launch_gp_append(r->gp.dev, kparams(r->cfg.kernel), r->cfg.noise, r->space->dev(), -1, r->d_xnew, y_raw, n0,
                       nullptr, r->stream);
      GTC_LAUNCHED();
      const VarPartials vp = r->vp();
      launch_extend(r->space->dev(), r->gp.dev, kparams(r->cfg.kernel), r->V, r->tile_stride, n0, 1, true, r->mu,
                    r->var, true, &vp, r->tstat, r->stream);
      GTC_LAUNCHED();
      r->acc_valid = true;
      r->predictions_valid = true;
      appended = true;
    }
  }
  if ((rc = enqueue_local_totals(r))) return rc;
  GTC_CUDA(cudaMemcpyAsync(r->red.h_totals, r->red.totals, sizeof(VarTotals), cudaMemcpyDeviceToHost, r->stream));
  GTC_CUDA(cudaMemcpyAsync(&r->h_rb->sc, r->gp.dev.sc, sizeof(GpScalars), cudaMemcpyDeviceToHost, r->stream));
  GTC_CUDA(cudaStreamSynchronize(r->stream));
  if (appended) {
    if (r->h_rb->sc.status != 0) {  // bordered pivot <= 0: escalate exactly like a refit (gp.hpp:116-129)
      if ((rc = refit(r, r->jitter * 2.0, info))) return rc;
      if ((rc = enqueue_local_totals(r))) return rc;
      GTC_CUDA(cudaMemcpyAsync(r->red.h_totals, r->red.totals, sizeof(VarTotals), cudaMemcpyDeviceToHost, r->stream));
      GTC_CUDA(cudaStreamSynchronize(r->stream));
    } else {
      r->n = n0 + 1;
      *r->gp.h_sc = r->h_rb->sc;
      fill_info(info, r->h_rb->sc, r->n, 0);
    }
  } else if (!valid) {
    fill_info(info, *r->gp.h_sc, r->n, 0);
  }
  *var_sum = r->red.h_totals->sum;
  *var_count = r->red.h_totals->count;
  return GTC_OK;
}

extern "C" int gtc_shard_select(gtc_run* r, const gtc_select_args* a, double global_var_sum,
                                int64_t global_var_count, gtc_shard_selection* out) {
  if (!r || !a || !out) return fail(GTC_ERR_INVALID, "null argument");
  if ((a->af_mask & 7u) == 0) return fail(GTC_ERR_INVALID, "af_mask selects no acquisition function");
  GTC_CUDA(cudaSetDevice(r->space->device));
  // global -> local exclusions (only those on this shard)
  std::vector<int64_t> local_ex;
  for (int32_t k = 0; k < a->n_excluded; ++k) {
    const int64_t p = a->excluded[k] - r->shard_offset;
    if (p >= 0 && p < r->space->n) local_ex.push_back(p);
  }
  gtc_select_args la = *a;
  la.excluded = local_ex.empty() ? nullptr : local_ex.data();
  la.n_excluded = (int32_t)local_ex.size();
  int rc = enqueue_selection(r, &la, true, global_var_sum, (long long)global_var_count);  // totals by value
  if (rc) return rc;
  GTC_CUDA(cudaMemcpyAsync(r->red.h_sel, r->red.sel, sizeof(SelectDev), cudaMemcpyDeviceToHost, r->stream));
  GTC_CUDA(cudaStreamSynchronize(r->stream));
  const SelectDev& s = *r->red.h_sel;
  const int64_t off = r->shard_offset;
  for (int k = 0; k < 3; ++k) {
    out->best_position[k] = s.best_nonnan_pos[k] >= 0 ? s.best_nonnan_pos[k] + off : -1;
    out->best_score[k] = s.best_nonnan_score[k];
  }
  out->first_eligible = s.first_eligible >= 0 ? s.first_eligible + off : -1;
  out->first_nan_mask = s.n_candidates > 0 ? s.first_nan_mask : 0u;
  out->n_candidates = s.n_candidates;
  out->lambda = s.lambda;
  out->mean_variance = s.mean_variance;
  out->best_std = s.best_std;
  out->cv_fallback = s.cv_fallback;
  return GTC_OK;
}

extern "C" int gtc_select(gtc_run* r, const gtc_select_args* a, gtc_select_result* out) {
  if (!r || !a || !out) return fail(GTC_ERR_INVALID, "null argument");
  if ((a->af_mask & 7u) == 0) return fail(GTC_ERR_INVALID, "af_mask selects no acquisition function");
  GTC_CUDA(cudaSetDevice(r->space->device));
  int rc = enqueue_selection(r, a);
  if (rc) return rc;
  GTC_CUDA(cudaMemcpyAsync(r->red.h_sel, r->red.sel, sizeof(SelectDev), cudaMemcpyDeviceToHost, r->stream));
  GTC_CUDA(cudaStreamSynchronize(r->stream));
  copy_result(*r->red.h_sel, out);
  if (r->red.h_sel->n_candidates == 0) return fail(GTC_ERR_NO_CANDIDATES, "acquisition: no candidates remaining");
  return GTC_OK;
}

// One BO iteration's device work after an evaluation, with a single host
// synchronisation: mark visited -> (valid) bordered row + V-row pass ->
// (optional) cooperative selection -> one readback.  A failed bordered pivot
// is detected on the device (the pass is skipped, the selection reports
// GpScalars::status) and handled here by the escalating refit.
// One gtc_observe call, split so that a group can run the device part of
// many runs' calls in shared launches (gtc_run_bo_batch).
struct ObserveReq {
  gtc_run* r;
  int64_t pos;
  double y_raw;
  int32_t valid;
  const gtc_select_args* a;
  bool newly = false;
  int n0 = 0;
  bool appended = false;   // bordered append + pass enqueued
  bool selecting = false;  // selection enqueued
  int status = GTC_OK;     // device-phase failure
  std::string error;
  std::binary_semaphore done{0};  // released by the group's executor
};

// Host bookkeeping before the device work.
static void observe_prepare(ObserveReq& q) {
  gtc_run* r = q.r;
  q.newly = host_mark(r, q.pos, 1);
  q.n0 = r->n;
  if (q.valid) {
    keep_obs(r, q.n0);
    push_obs(r, &r->space->host_coords[(size_t)q.pos * r->space->d], q.y_raw);
  }
}

// The device part on the run's own stream (single-run path).
static int observe_device(ObserveReq& q, gtc_fit_info* info) {
  gtc_run* r = q.r;
  int rc;
  if (!(q.valid && q.n0 > 0) && (rc = flush_stats(r))) return rc;  // (an append recomputes them)
  set_thread_pdl(r->pdl);
  const bool ev = phase_events();
  if (ev) GTC_CUDA(cudaEventRecord(r->ev_step0, r->stream));
  if (q.valid) {
    if (q.n0 == 0) {
      if (q.newly) {
        launch_mark(r->visited, q.pos, 1, r->stream);
        GTC_LAUNCHED();
        r->acc_valid = false;
      }
      if ((rc = refit(r, r->cfg.jitter, info))) return rc;
    } else {
      if ((rc = enqueue_append(r, q.pos, q.y_raw, q.newly ? r->visited : nullptr))) return rc;
      r->predictions_valid = true;
      q.appended = true;
    }
  } else if (q.newly) {
    VarAccum* acc = r->live_acc();
    launch_mark(r->visited, q.pos, 1, r->stream, acc, r->var, r->cfg.kernel.output_variance);
    GTC_LAUNCHED();
    r->acc_valid = acc != nullptr;
  }
  q.selecting = q.a && r->space->n - r->visited_count > 0;
  // direct read-back: the selection's last block writes its record and the
  // GP scalars into the pinned h_rb and then a sequence word the host spins
  // on -- no copy-engine transfers and no stream synchronisation on the
  // iteration's critical path (phase events keep the synchronising path)
  const bool direct = q.selecting && !ev;
  const uint32_t seq = direct ? ++r->rb_seq : 0;
  if (q.selecting && (rc = enqueue_selection(r, q.a, false, 0.0, 0, seq))) return rc;
  if (ev) GTC_CUDA(cudaEventRecord(r->ev_step1, r->stream));
  r->step_timed = ev;
  r->step_appended = q.appended;
  if (direct) {
    const volatile uint32_t* flag = &r->h_rb->seq;
    for (uint32_t spins = 0; *flag != seq; ++spins) {
      if ((spins & 1023u) == 1023u) {  // the stream finished (or failed) without the flag?
        const cudaError_t e = cudaStreamQuery(r->stream);
        if (e != cudaErrorNotReady) {
          if (e != cudaSuccess) GTC_CUDA(e);
          if (*flag != seq) return fail(GTC_ERR_CUDA, "selection finished without its read-back");
          break;
        }
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return GTC_OK;
  }
  if (q.selecting)
    GTC_CUDA(cudaMemcpyAsync(&r->h_rb->sel, r->red.sel, sizeof(SelectDev), cudaMemcpyDeviceToHost, r->stream));
  GTC_CUDA(cudaMemcpyAsync(&r->h_rb->sc, r->gp.dev.sc, sizeof(GpScalars), cudaMemcpyDeviceToHost, r->stream));
  GTC_CUDA(cudaStreamSynchronize(r->stream));
  return GTC_OK;
}

// After the device work (h_rb holds the scalars and the selection).
static int observe_finish(ObserveReq& q, gtc_select_result* out, gtc_fit_info* info) {
  gtc_run* r = q.r;
  int rc;
  if (q.appended) {
    if (r->h_rb->sc.status != 0) {
      // bordered pivot <= 0: refactorise with escalated jitter (gp.hpp:116-129)
      if ((rc = refit(r, r->jitter * 2.0, info))) return rc;
      if (q.selecting) {
        if ((rc = enqueue_selection(r, q.a))) return rc;
        GTC_CUDA(cudaMemcpyAsync(&r->h_rb->sel, r->red.sel, sizeof(SelectDev), cudaMemcpyDeviceToHost, r->stream));
        GTC_CUDA(cudaStreamSynchronize(r->stream));
      }
    } else {
      r->n = q.n0 + 1;
      *r->gp.h_sc = r->h_rb->sc;
      fill_info(info, r->h_rb->sc, r->n, 0);
    }
  } else if (!q.valid) {
    fill_info(info, r->h_rb->sc, r->n, 0);
  }
  if (q.selecting && out) {
    copy_result(r->h_rb->sel, out);
    if (r->h_rb->sel.n_candidates == 0) return fail(GTC_ERR_NO_CANDIDATES, "acquisition: no candidates remaining");
  } else if (out) {
    std::memset(out, 0, sizeof(*out));
    for (int k = 0; k < 3; ++k) out->position[k] = -1;
  }
  return GTC_OK;
}

// ---- observe groups (gtc_run_bo_batch) -------------------------------------
// The member threads of a group each drive their own run; a gtc_observe of a
// grouped run queues its request and waits until every member has queued
// one (or left), then the last one to arrive enqueues the device work of all
// queued requests in shared launches on the group's stream -- marks, one
// bordered-append launch, one predictive-pass launch, one selection launch
// per AF mask -- and one read-back.  Results are bit-identical to the
// single-run path (same kernels, same per-run arguments).
struct gtc_group {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  int members = 0;
  std::atomic<uint64_t> round{0};  // completed rounds (waiters spin on it, no lock hand-off)
  std::vector<ObserveReq*> queue;
  unsigned char* h_buf = nullptr;  // pinned staging (arguments, results)
  unsigned char* d_buf = nullptr;
  size_t cap = 0;
  // diagnostics (GTC_GROUP_STATS=1 prints them at destroy)
  uint64_t n_rounds = 0, n_requests = 0;
  double t_exec = 0.0, t_first = -1.0, t_last = 0.0, t_enqueued = 0.0, t_round0 = 0.0;
};

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static int group_reserve(gtc_group* g, size_t bytes) {
  if (bytes <= g->cap) return GTC_OK;
  const size_t cap = std::max(bytes, 2 * g->cap);
  if (g->h_buf) cudaFreeHost(g->h_buf);
  if (g->d_buf) cudaFree(g->d_buf);
  g->h_buf = g->d_buf = nullptr;
  g->cap = 0;
  GTC_CUDA(cudaMallocHost(&g->h_buf, cap));
  GTC_CUDA(cudaMalloc(&g->d_buf, cap));
  g->cap = cap;
  return GTC_OK;
}

static size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

// Device work of every queued request (called with the group lock held).
static int execute_round(gtc_group* g) {
  std::vector<ObserveReq*>& Q = g->queue;
  const int R = (int)Q.size();
  GTC_CUDA(cudaSetDevice(g->device));
  std::vector<cudaStream_t> saved(R);
  for (int i = 0; i < R; ++i) {  // every run's device work of this round on the group stream
    saved[i] = Q[i]->r->stream;
    Q[i]->r->stream = g->stream;
  }
  struct Restore {
    std::vector<ObserveReq*>& Q;
    std::vector<cudaStream_t>& saved;
    ~Restore() {
      for (size_t i = 0; i < Q.size(); ++i) Q[i]->r->stream = saved[i];
    }
  } restore{Q, saved};
  // layout of the staging buffer
  const size_t o_app = 0, o_ext = align16(o_app + sizeof(AppendArgs) * R);
  const size_t o_sel = align16(o_ext + sizeof(ExtendArgs) * R), o_mark = align16(o_sel + sizeof(SelectRunArgs) * R);
  const size_t o_gat = align16(o_mark + sizeof(MarkDesc) * R), o_res = align16(o_gat + sizeof(GatherDesc) * 2 * R);
  const size_t per_res = align16(sizeof(SelectDev)) + align16(sizeof(GpScalars));
  // (+ one masked copy of the selection arguments per AF mask, for rounds
  // whose runs ask for different AF sets)
  const size_t o_msk = align16(o_res + per_res * R);
  int rc = group_reserve(g, o_msk + sizeof(SelectRunArgs) * R * 8);
  if (rc) return rc;
  auto* app = reinterpret_cast<AppendArgs*>(g->h_buf + o_app);
  auto* ext = reinterpret_cast<ExtendArgs*>(g->h_buf + o_ext);
  auto* sel = reinterpret_cast<SelectRunArgs*>(g->h_buf + o_sel);
  auto* mark = reinterpret_cast<MarkDesc*>(g->h_buf + o_mark);
  auto* gat = reinterpret_cast<GatherDesc*>(g->h_buf + o_gat);
  // 1. marks of invalid evaluations, appends + passes of valid ones
  int n_mark = 0, n_app = 0, nu = -1, max_n0 = 0, d = 0;
  size_t app_smem = 0;
  int64_t tiles = 0, n_cand = 0;
  for (int i = 0; i < R; ++i) {
    ObserveReq& q = *Q[i];
    gtc_run* r = q.r;
    app[i] = AppendArgs{};
    ext[i] = ExtendArgs{};
    sel[i] = SelectRunArgs{};
    d = r->space->d;
    tiles = r->space->n_pad / kTile;
    n_cand = r->space->n;
    if (q.valid) {
      size_t sm;
      r->stats_stale = -1;  // (the bordered row recomputes the standardisation and beta)
      app[i] = make_append_args(r->gp.dev, kparams(r->cfg.kernel), r->cfg.noise, r->space->dev(), q.pos, nullptr,
                                q.y_raw, q.n0, q.newly ? r->visited : nullptr, &sm);
      app[i].V = r->V;  // bordered row from the pick's V column (exact substitution below the margin)
      app[i].tile_stride = r->tile_stride;
      const VarPartials vp = r->vp();
      ext[i] = make_pass_args(r->space->dev(), r->gp.dev, kparams(r->cfg.kernel), r->V, r->tile_stride, q.n0, r->mu,
                              r->var, &vp, r->tstat);
      app_smem = std::max(app_smem, sm);
      max_n0 = std::max(max_n0, q.n0);
      nu = r->cfg.kernel.nu;
      r->acc_valid = true;
      r->predictions_valid = true;
      r->pass_timed = false;
      q.appended = true;
      ++n_app;
    } else if (q.newly) {
      VarAccum* acc = r->live_acc();
      mark[n_mark++] = MarkDesc{r->visited, q.pos, acc, r->var, r->cfg.kernel.output_variance};
      r->acc_valid = acc != nullptr;
    }
    r->step_timed = false;
  }
  // arguments of the append / pass / mark launches: one copy
  GTC_CUDA(cudaMemcpyAsync(g->d_buf, g->h_buf, o_sel, cudaMemcpyHostToDevice, g->stream));
  if (n_mark) {
    GTC_CUDA(cudaMemcpyAsync(g->d_buf + o_mark, g->h_buf + o_mark, sizeof(MarkDesc) * n_mark, cudaMemcpyHostToDevice,
                             g->stream));
    launch_mark_batch(reinterpret_cast<MarkDesc*>(g->d_buf + o_mark), n_mark, g->stream);
    GTC_LAUNCHED();
  }
  if (n_app) {
    launch_gp_append_batch(reinterpret_cast<AppendArgs*>(g->d_buf + o_app), R, nu, app_smem, g->stream);
    GTC_LAUNCHED();
    launch_extend_batch(reinterpret_cast<ExtendArgs*>(g->d_buf + o_ext), R, tiles, nu, max_n0, d, g->stream);
    GTC_LAUNCHED();
  }
  // 2. selections (auxiliary per-run work -- exclusions, variance totals after
  // marks -- is enqueued on the group stream by build_selection)
  uint32_t masks = 0;
  for (int i = 0; i < R; ++i) {
    ObserveReq& q = *Q[i];
    q.selecting = q.a && q.r->space->n - q.r->visited_count > 0;
    if (!q.selecting) continue;
    if ((rc = build_selection(q.r, q.a, false, 0.0, 0, &sel[i]))) {
      q.status = rc;
      q.error = g_last_error;
      q.selecting = false;
      sel[i] = SelectRunArgs{};
      continue;
    }
    masks |= 1u << (sel[i].p.af_mask & 7u);
  }
  if (masks) {
    GTC_CUDA(cudaMemcpyAsync(g->d_buf + o_sel, g->h_buf + o_sel, sizeof(SelectRunArgs) * R, cudaMemcpyHostToDevice,
                             g->stream));
    for (uint32_t m = 1; m < 8; ++m) {
      if (!(masks & (1u << m))) continue;
      // one launch per mask: runs with another mask see out == nullptr
      if (masks == (1u << m)) {
        launch_select_batch(reinterpret_cast<SelectRunArgs*>(g->d_buf + o_sel), R, m, n_cand, g->stream);
      } else {  // mixed masks: a masked copy of the argument array per mask
        const size_t off = o_msk + sizeof(SelectRunArgs) * R * m;
        auto* hs = reinterpret_cast<SelectRunArgs*>(g->h_buf + off);
        for (int i = 0; i < R; ++i) {
          hs[i] = sel[i];
          if ((sel[i].p.af_mask & 7u) != m) hs[i].out = nullptr;
        }
        GTC_CUDA(cudaMemcpyAsync(g->d_buf + off, hs, sizeof(SelectRunArgs) * R, cudaMemcpyHostToDevice, g->stream));
        launch_select_batch(reinterpret_cast<SelectRunArgs*>(g->d_buf + off), R, m, n_cand, g->stream);
      }
      GTC_LAUNCHED();
    }
  }
  // 3. one read-back of every run's selection record and GP scalars
  int n_gat = 0;
  for (int i = 0; i < R; ++i) {
    ObserveReq& q = *Q[i];
    const uint32_t base = (uint32_t)(per_res * i);
    if (q.selecting)
      gat[n_gat++] = GatherDesc{reinterpret_cast<const unsigned char*>(q.r->red.sel), (uint32_t)sizeof(SelectDev), base};
    gat[n_gat++] = GatherDesc{reinterpret_cast<const unsigned char*>(q.r->gp.dev.sc), (uint32_t)sizeof(GpScalars),
                              base + (uint32_t)align16(sizeof(SelectDev))};
  }
  GTC_CUDA(cudaMemcpyAsync(g->d_buf + o_gat, g->h_buf + o_gat, sizeof(GatherDesc) * n_gat, cudaMemcpyHostToDevice,
                           g->stream));
  launch_gather(reinterpret_cast<GatherDesc*>(g->d_buf + o_gat), n_gat, g->d_buf + o_res, g->stream);
  GTC_LAUNCHED();
  GTC_CUDA(cudaMemcpyAsync(g->h_buf + o_res, g->d_buf + o_res, per_res * R, cudaMemcpyDeviceToHost, g->stream));
  g->t_enqueued += now_s() - g->t_round0;
  GTC_CUDA(cudaStreamSynchronize(g->stream));
  for (int i = 0; i < R; ++i) {
    ObserveReq& q = *Q[i];
    const unsigned char* base = g->h_buf + o_res + per_res * i;
    if (q.selecting) std::memcpy(&q.r->h_rb->sel, base, sizeof(SelectDev));
    std::memcpy(&q.r->h_rb->sc, base + align16(sizeof(SelectDev)), sizeof(GpScalars));
  }
  return GTC_OK;
}

static int group_observe(ObserveReq& q, gtc_fit_info*) {
  gtc_group* g = q.r->group;
  std::unique_lock<std::mutex> lk(g->mu);
  g->queue.push_back(&q);
  const uint64_t my_round = g->round.load(std::memory_order_relaxed);
  if ((int)g->queue.size() >= g->members) {
    const double t0 = now_s();
    g->t_round0 = t0;
    const int rc = execute_round(g);
    const double t1 = now_s();
    g->t_exec += t1 - t0;
    ++g->n_rounds;
    g->n_requests += g->queue.size();
    if (g->t_first < 0) g->t_first = t0;
    g->t_last = t1;
    if (rc)
      for (ObserveReq* o : g->queue)
        if (!o->status) {
          o->status = rc;
          o->error = g_last_error;
        }
    g->round.fetch_add(1, std::memory_order_release);
    for (ObserveReq* o : g->queue)
      if (o != &q) o->done.release();  // one wake-up per waiter, no shared lock hand-off
    g->queue.clear();
  } else {
    lk.unlock();
    // a short spin catches quick rounds; then sleep on this request's semaphore
    for (int spin = 0; spin < 32 && g->round.load(std::memory_order_acquire) == my_round; ++spin)
      std::this_thread::yield();
    q.done.acquire();
  }
  if (q.status) return fail(q.status, q.error);
  return GTC_OK;
}

extern "C" int gtc_group_create(int device, gtc_group** out) {
  if (!out) return fail(GTC_ERR_INVALID, "out is null");
  GTC_CUDA(cudaSetDevice(device));
  auto* g = new gtc_group();
  g->device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete g;
    return fail(GTC_ERR_CUDA, std::string("group stream: ") + cudaGetErrorString(e));
  }
  *out = g;
  return GTC_OK;
}

extern "C" int gtc_group_destroy(gtc_group* g) {
  if (!g) return GTC_OK;
  if (std::getenv("GTC_GROUP_STATS"))
    std::fprintf(stderr, "gtc_group: %llu rounds, %.1f requests/round, host enqueue %.1f, exec %.1f us/round, span %.1f us/round\n",
                 (unsigned long long)g->n_rounds, g->n_rounds ? (double)g->n_requests / g->n_rounds : 0.0,
                 g->n_rounds ? 1e6 * g->t_enqueued / g->n_rounds : 0.0,
                 g->n_rounds ? 1e6 * g->t_exec / g->n_rounds : 0.0,
                 g->n_rounds ? 1e6 * (g->t_last - g->t_first) / g->n_rounds : 0.0);
  cudaSetDevice(g->device);
  cudaStreamSynchronize(g->stream);
  cudaStreamDestroy(g->stream);
  if (g->h_buf) cudaFreeHost(g->h_buf);
  if (g->d_buf) cudaFree(g->d_buf);
  delete g;
  return GTC_OK;
}

extern "C" int gtc_group_join(gtc_group* g) {
  if (!g) return fail(GTC_ERR_INVALID, "group is null");
  std::lock_guard<std::mutex> lk(g->mu);
  ++g->members;
  return GTC_OK;
}

extern "C" int gtc_group_leave(gtc_group* g) {
  if (!g) return fail(GTC_ERR_INVALID, "group is null");
  std::lock_guard<std::mutex> lk(g->mu);
  --g->members;
  if (!g->queue.empty() && (int)g->queue.size() >= g->members) {  // the rest are all waiting
    g->t_round0 = now_s();
    const int rc = execute_round(g);
    if (rc)
      for (ObserveReq* o : g->queue)
        if (!o->status) {
          o->status = rc;
          o->error = g_last_error;
        }
    g->round.fetch_add(1, std::memory_order_release);
    for (ObserveReq* o : g->queue) o->done.release();
    g->queue.clear();
  }
  return GTC_OK;
}

extern "C" int gtc_run_set_group(gtc_run* r, gtc_group* g) {
  if (!r) return fail(GTC_ERR_INVALID, "run is null");
  if (g && g->device != r->space->device) return fail(GTC_ERR_INVALID, "group and run are on different devices");
  r->group = g;
  return GTC_OK;
}

extern "C" int gtc_observe(gtc_run* r, int64_t pos, double y_raw, int32_t valid, const gtc_select_args* a,
                           gtc_select_result* out, gtc_fit_info* info) {
  if (!r) return fail(GTC_ERR_INVALID, "run is null");
  if (pos < 0 || pos >= r->space->n) return fail(GTC_ERR_INVALID, "position out of range");
  if (valid && !std::isfinite(y_raw)) return fail(GTC_ERR_INVALID, "GP fit: observations must be finite");
  if (valid && r->n >= r->cfg.n_max) return fail(GTC_ERR_CAPACITY, "more observations than the run's n_max");
  if (a && (a->af_mask & 7u) == 0) return fail(GTC_ERR_INVALID, "af_mask selects no acquisition function");
  GTC_CUDA(cudaSetDevice(r->space->device));
  ObserveReq q{r, pos, y_raw, valid, a};
  observe_prepare(q);
  // the first observation refits from scratch: always on the run's own stream
  const int rc = (r->group && !(q.valid && q.n0 == 0)) ? group_observe(q, info) : observe_device(q, info);
  if (rc) return rc;
  return observe_finish(q, out, info);
}

extern "C" int gtc_read_predictions(gtc_run* r, double* mean, double* variance) {
  if (!r) return fail(GTC_ERR_INVALID, "run is null");
  GTC_CUDA(cudaSetDevice(r->space->device));
  int rc = ensure_predictions(r);
  if (rc) return rc;
  if (mean) GTC_CUDA(cudaMemcpyAsync(mean, r->mu, sizeof(double) * r->space->n, cudaMemcpyDeviceToHost, r->stream));
  if (variance) GTC_CUDA(cudaMemcpyAsync(variance, r->var, sizeof(double) * r->space->n, cudaMemcpyDeviceToHost, r->stream));
  GTC_CUDA(cudaStreamSynchronize(r->stream));
  return GTC_OK;
}

static double event_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventSynchronize(b) != cudaSuccess) return 0.0;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) return 0.0;
  return ms;
}

extern "C" double gtc_last_pass_ms(const gtc_run* r) {
  return r && r->pass_timed ? event_ms(r->ev0, r->ev1) : 0.0;
}
extern "C" double gtc_last_step_ms(const gtc_run* r) {
  return r && r->step_timed ? event_ms(r->ev_step0, r->ev_step1) : 0.0;
}
extern "C" int gtc_last_phase_ms(const gtc_run* r, double* out) {
  if (!r || !out) return fail(GTC_ERR_INVALID, "null argument");
  if (!r->step_timed || !r->pass_timed || !r->step_appended) return fail(GTC_ERR_INVALID, "last observe did not append");
  out[0] = event_ms(r->ev_step0, r->ev0);
  out[1] = event_ms(r->ev0, r->ev1);
  out[2] = event_ms(r->ev1, r->ev_step1);
  return GTC_OK;
}
extern "C" int gtc_debug_append_marks(const gtc_run* r, uint64_t* marks) {
  if (!r || !marks) return fail(GTC_ERR_INVALID, "null argument");
  for (int i = 0; i < 7; ++i) marks[i] = r->h_rb->sc.t[i];
  return GTC_OK;
}

extern "C" int gtc_debug_select_trace(uint64_t* marks, int32_t rows) {
  if (!marks || rows <= 0 || rows > 2048) return fail(GTC_ERR_INVALID, "bad arguments");
  if (read_sel_trace(reinterpret_cast<unsigned long long*>(marks), rows))
    return fail(GTC_ERR_INVALID, "library built without GTC_SEL_TRACE");
  return GTC_OK;
}

extern "C" int gtc_debug_set_rebuild(int32_t mode) {
  const int prev = rebuild_mode();
  if (mode >= 0) set_rebuild_mode(mode > 4 ? 4 : mode);
  return prev;
}

extern "C" int gtc_debug_set_factor(int32_t mode) {
  const int prev = factor_mode();
  if (mode >= 0) set_factor_mode(mode ? 1 : 0);
  return prev;
}

extern "C" int64_t gtc_run_exact_rows(const gtc_run* r) { return r ? (int64_t)r->gp.h_sc->exact_rows : -1; }
extern "C" uint64_t gtc_run_stream(const gtc_run* r) { return r ? (uint64_t)(uintptr_t)r->stream : 0; }

// =============================================================== stand-alone GpModel

extern "C" int gtc_gp_destroy(gtc_gp* g) {
  if (!g) return GTC_OK;
  cudaSetDevice(g->device);
  if (g->stream) cudaStreamSynchronize(g->stream);
  g->gp.release();
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
  return GTC_OK;
}

extern "C" int gtc_gp_fit(int device, const gtc_kernel* kernel, const double* X, const double* y,
                          int32_t n, int32_t d, double noise, double jitter, gtc_gp** out,
                          gtc_fit_info* info) {
  if (!out) return fail(GTC_ERR_INVALID, "out is null");
  *out = nullptr;
  int rc = check_kernel(kernel);
  if (rc) return rc;
  if ((rc = check_fit_inputs(y, n, noise, jitter))) return rc;
  if (d <= 0 || d > kMaxDim) return fail(GTC_ERR_INVALID, "dimension out of range [1, 64]");
  if (n > kMaxNmax) return fail(GTC_ERR_CAPACITY, "more than 1024 observations");
  GTC_CUDA(cudaSetDevice(device));
  auto* g = new gtc_gp();
  g->device = device;
  g->kernel = *kernel;
  g->noise = noise;
  g->jitter = jitter;
  g->n = n;
  g->d = d;
  if ((rc = g->gp.init(n > 0 ? n : 1, d))) {
    gtc_gp_destroy(g);
    return rc;
  }
  cudaError_t e = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    gtc_gp_destroy(g);
    return fail(GTC_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(e));
  }
  if (n > 0) {
    e = cudaMemcpyAsync(g->gp.dev.train_x, X, sizeof(double) * n * d, cudaMemcpyHostToDevice, g->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->gp.dev.y, y, sizeof(double) * n, cudaMemcpyHostToDevice, g->stream);
    if (e != cudaSuccess) {
      gtc_gp_destroy(g);
      return fail(GTC_ERR_CUDA, std::string("upload: ") + cudaGetErrorString(e));
    }
    rc = factor_with_escalation(g->gp, g->kernel, noise, jitter, jitter, n, g->stream);
    if (rc) {
      const std::string msg = g_last_error;
      gtc_gp_destroy(g);
      return fail(rc, msg);
    }
  } else {
    g->gp.h_sc->jitter = jitter;
  }
  fill_info(info, *g->gp.h_sc, n, 1);
  *out = g;
  return GTC_OK;
}

extern "C" int gtc_gp_predict(gtc_gp* g, const double* Xstar, int64_t m, double* mean, double* variance) {
  if (!g) return fail(GTC_ERR_INVALID, "gp is null");
  if (m < 0) return fail(GTC_ERR_INVALID, "negative point count");
  if (m == 0) return GTC_OK;
  GTC_CUDA(cudaSetDevice(g->device));
  gtc_space* sp = nullptr;
  int rc = gtc_space_create(g->device, Xstar, m, g->d, &sp);
  if (rc) return rc;
  const int64_t tiles = sp->n_pad / kTile;
  const int64_t tile_stride = (int64_t)(g->n > 0 ? g->n : 1) * kTile;
  double *V = nullptr, *mu = nullptr, *var = nullptr;
  if ((rc = dalloc(&V, (size_t)tiles * tile_stride)) || (rc = dalloc(&mu, sp->n_pad)) ||
      (rc = dalloc(&var, sp->n_pad))) {
    cudaFree(V); cudaFree(mu); cudaFree(var);
    gtc_space_destroy(sp);
    return rc;
  }
  // GpDev with n_max = n so the extend kernel's tile stride matches the factor
  rc = rebuild_predictions(sp->dev(), g->gp, g->kernel, V, tile_stride, g->n, mu, var, nullptr, nullptr, g->stream);
  cudaError_t e = cudaSuccess;
  if (!rc && mean) e = cudaMemcpyAsync(mean, mu, sizeof(double) * m, cudaMemcpyDeviceToHost, g->stream);
  if (!rc && e == cudaSuccess && variance) e = cudaMemcpyAsync(variance, var, sizeof(double) * m, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  cudaFree(V); cudaFree(mu); cudaFree(var);
  gtc_space_destroy(sp);
  if (rc) return rc;
  if (e != cudaSuccess) return fail(GTC_ERR_CUDA, std::string("predict: ") + cudaGetErrorString(e));
  return GTC_OK;
}

extern "C" int gtc_gp_info(const gtc_gp* g, gtc_fit_info* info) {
  if (!g || !info) return fail(GTC_ERR_INVALID, "null argument");
  fill_info(info, *g->gp.h_sc, g->n, 1);
  return GTC_OK;
}

// =============================================================== acquisition over spans

extern "C" int gtc_best_candidate(int device, int32_t af, const double* means, const double* stds,
                                  int64_t n, double best_std, double lambda, const uint8_t* excluded,
                                  int64_t* position_out, double* score_out) {
  if (af < 0 || af > 2) return fail(GTC_ERR_INVALID, "unknown acquisition function");
  if (n <= 0) return fail(GTC_ERR_NO_CANDIDATES, "acquisition: no candidates remaining");
  GTC_CUDA(cudaSetDevice(device));
  cudaStream_t s;
  GTC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  ReduceScratch red;
  double *dm = nullptr, *ds = nullptr;
  uint8_t* dx = nullptr;
  int rc = red.init(n);
  if (!rc) rc = dalloc(&dm, n);
  if (!rc) rc = dalloc(&ds, n);
  if (!rc && excluded) rc = dalloc(&dx, n);
  cudaError_t e = cudaSuccess;
  if (!rc) {
    e = cudaMemcpyAsync(dm, means, sizeof(double) * n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ds, stds, sizeof(double) * n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && excluded) e = cudaMemcpyAsync(dx, excluded, n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
      launch_best_candidate(dm, ds, dx, n, af, best_std, lambda, red.b, red.sel, s);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(red.h_sel, red.sel, sizeof(SelectDev), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  SelectDev res{};
  if (!rc && e == cudaSuccess) res = *red.h_sel;
  cudaFree(dm); cudaFree(ds); cudaFree(dx);
  red.release();
  cudaStreamDestroy(s);
  if (rc) return rc;
  if (e != cudaSuccess) return fail(GTC_ERR_CUDA, std::string("best_candidate: ") + cudaGetErrorString(e));
  if (res.n_candidates == 0) return fail(GTC_ERR_NO_CANDIDATES, "acquisition: no candidates remaining");
  if (position_out) *position_out = res.position[af];
  if (score_out) *score_out = res.score[af];
  return GTC_OK;
}

extern "C" int gtc_acquisition_scores(int device, int32_t af, const double* means, const double* stds,
                                      int64_t n, double best_std, double lambda, double* scores_out) {
  if (af < 0 || af > 2) return fail(GTC_ERR_INVALID, "unknown acquisition function");
  if (n <= 0) return GTC_OK;
  GTC_CUDA(cudaSetDevice(device));
  cudaStream_t s;
  GTC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double *dm = nullptr, *ds = nullptr, *dout = nullptr;
  int rc = dalloc(&dm, n);
  if (!rc) rc = dalloc(&ds, n);
  if (!rc) rc = dalloc(&dout, n);
  cudaError_t e = cudaSuccess;
  if (!rc) {
    e = cudaMemcpyAsync(dm, means, sizeof(double) * n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ds, stds, sizeof(double) * n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
      launch_scores(dm, ds, n, af, best_std, lambda, dout, s);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(scores_out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  cudaFree(dm); cudaFree(ds); cudaFree(dout);
  cudaStreamDestroy(s);
  if (rc) return rc;
  if (e != cudaSuccess) return fail(GTC_ERR_CUDA, std::string("acquisition_scores: ") + cudaGetErrorString(e));
  return GTC_OK;
}
