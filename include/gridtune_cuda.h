/*
 * gridtune_cuda.h — C ABI of the B200-native BO surrogate pass.
 *
 * Drop-in boundary for the per-iteration surrogate pass of the reference
 * `gridtune` BO tuner (/root/reference/proj/include/gridtune).  The reference
 * binds this path as header-only C++ (no FFI); every entry point below replaces
 * one reference call site, cited as file:line.  INTEGRATION.md shows the
 * reference-side binding.  Plain pointers and sizes only; no torch / CUDA types.
 *
 * Conventions
 *  - All arithmetic is IEEE FP64; positions are int64 indices into the
 *    caller's enumerated candidate list (EnumeratedSpace::configs order,
 *    search_space.hpp:216-245), ascending canonical index.
 *  - Host buffers are caller-owned and only read/written during the call.
 *    Device memory is owned by the handle.
 *  - Status: 0 = OK, negative = error (mapped to gridtune exception types by
 *    the C++ host layer, errors.hpp:55-108).  gtc_last_error() returns the
 *    message of the last failing call on the calling thread.
 *  - Re-entrant per handle: no global mutable state; each run owns one CUDA
 *    stream; distinct handles may be used from different host threads and
 *    devices concurrently (experiment.hpp:335-358 runs BO runs in a pool).
 *  - There is no CPU fallback: every compute entry point runs sm_100a kernels
 *    and fails with GTC_ERR_CUDA when no device is usable.
 */
#ifndef GRIDTUNE_CUDA_H_
#define GRIDTUNE_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (C++ exception each maps to) --------------------------- */
#define GTC_OK 0
#define GTC_ERR_INVALID (-1)       /* gridtune::Error (bad argument, "GP fit: ...")   */
#define GTC_ERR_CONDITIONING (-2)  /* gridtune::ModelConditioningError, gp.hpp:123-127 */
#define GTC_ERR_NO_CANDIDATES (-3) /* Error("acquisition: no candidates remaining"),  portfolio.hpp:57-59 */
#define GTC_ERR_CUDA (-4)          /* CUDA runtime failure / no device                */
#define GTC_ERR_OOM (-5)           /* device allocation failed                         */
#define GTC_ERR_CONFIG (-6)        /* gridtune::ConfigError                            */
#define GTC_ERR_CAPACITY (-7)      /* more observations than the run's n_max          */
#define GTC_ERR_SAMPLING (-8)      /* gridtune::SamplingError (run_bo preconditions, initial design) */
#define GTC_ERR_ABORTED (-9)       /* the objective callback asked to stop            */
#define GTC_ERR_PARSE (-10)        /* gridtune::ParseError (restriction syntax / types), errors.hpp:17-26 */
#define GTC_ERR_EMPTY (-11)        /* gridtune::EmptySearchSpaceError, errors.hpp:29-32 */

/* ---- enums mirroring the reference ---------------------------------------- */
/* MaternNu, gp.hpp:12 */
#define GTC_NU_HALF 0
#define GTC_NU_THREE_HALVES 1
#define GTC_NU_FIVE_HALVES 2
/* AcquisitionId order ei, poi, lcb (acquisition.hpp:44); bit k selects slot k */
#define GTC_AF_EI 0
#define GTC_AF_POI 1
#define GTC_AF_LCB 2
#define GTC_AF_MASK(af) (1u << (af))
/* ExplorationConfig::Mode, acquisition.hpp:55-59 */
#define GTC_LAMBDA_CONSTANT 0
#define GTC_LAMBDA_CONTEXTUAL_VARIANCE 1

typedef struct gtc_space gtc_space; /* resident normalised search space      */
typedef struct gtc_run gtc_run;     /* one BO run's resident surrogate state */
typedef struct gtc_gp gtc_gp;       /* stand-alone GpModel (arbitrary points) */
typedef struct gtc_group gtc_group; /* batched observe across runs (one per batch) */

/* MaternKernel, gp.hpp:27-56 */
typedef struct {
  int32_t nu;             /* GTC_NU_* */
  double lengthscale;     /* > 0 */
  double output_variance; /* > 0 */
} gtc_kernel;

/* GpModel::fit arguments (gp.hpp:81-83) plus the run's capacity. */
typedef struct {
  gtc_kernel kernel;
  double noise;  /* >= 0, default 1e-10 */
  double jitter; /* > 0,  default 1e-6  */
  int32_t n_max; /* maximum GP training size for the run (budget)  */
} gtc_model_config;

/* Model scalars after a fit/append (GpModel accessors gp.hpp:137-142). */
typedef struct {
  int32_t n;      /* train_size()                           */
  int32_t rebuilt;/* 1 if the call refactorised from scratch (jitter escalation) */
  double y_mean;  /* y_mean()                               */
  double y_std;   /* y_std()                                */
  double jitter;  /* jitter() actually used                 */
} gtc_fit_info;

/* One iteration's selection request (strategies.hpp:404-436). */
typedef struct {
  uint32_t af_mask;              /* GTC_AF_MASK(GTC_AF_EI) | ...; every active AF of `multi` */
  int32_t lambda_mode;           /* GTC_LAMBDA_*                                        */
  double lambda_constant;        /* ExplorationConfig::constant (0.01)                   */
  double cv_initial_sample_mean; /* ContextualVarianceState, acquisition.hpp:63-66       */
  double cv_initial_mean_variance;
  double f_best_raw;             /* run's best raw observation (strategies.hpp:409,424)  */
  const int64_t* excluded;       /* optional positions to skip (portfolio pending set)  */
  int32_t n_excluded;
} gtc_select_args;

typedef struct {
  int64_t position[3];  /* argmax per AF slot (ei, poi, lcb); -1 when not requested  */
  double score[3];      /* the winning score (LCB slot holds -lcb, portfolio.hpp:47) */
  double lambda;        /* exploration factor used                                   */
  double mean_variance; /* mean posterior variance over the candidates               */
  double best_std;      /* GpModel::standardize(f_best_raw)                          */
  int64_t n_candidates; /* unvisited, non-excluded candidates scored                 */
  int32_t cv_fallback;  /* 1: contextual variance undefined, constant used          */
} gtc_select_result;

/* ---- library ---------------------------------------------------------------- */
const char* gtc_last_error(void);
const char* gtc_version(void);
/* Number of kernels this library has launched in the calling process. */
uint64_t gtc_kernel_launches(void);

/* ---- resident search space (EnumeratedSpace, search_space.hpp:216-245) ------ */
/* coords: n x d row-major, as EnumeratedSpace::coords[pos][j]
 * (SearchSpace::normalize, search_space.hpp:158-166).  Stored on `device` as
 * structure-of-arrays [d][n_pad]. */
int gtc_space_create(int device, const double* coords, int64_t n, int32_t d, gtc_space** out);
int gtc_space_destroy(gtc_space* space);
int64_t gtc_space_size(const gtc_space* space);

/* ---- device search-space enumeration (SearchSpace, search_space.hpp:23-207) - */
/* ParameterDef (parameter.hpp:62-125): kind 0 numeric (numbers), 1 categorical
 * (strings), 2 boolean (booleans, 0/1); values in declaration order. */
#define GTC_PARAM_NUMERIC 0
#define GTC_PARAM_CATEGORICAL 1
#define GTC_PARAM_BOOLEAN 2
typedef struct {
  const char* name;
  int32_t kind;
  int32_t n_values;
  const double* numbers;
  const char* const* strings;
  const uint8_t* booleans;
} gtc_param_def;

/* SearchSpace(params, restriction_sources) + EnumeratedSpace (search_space.hpp:
 * 35-44, 120-166, 216-245) on the device: parses and type-checks every
 * restriction (GTC_ERR_PARSE, message "... (at position p)", the position in
 * *error_position when non-null), validates the parameters (GTC_ERR_INVALID),
 * enumerates the Cartesian grid (limit 20,000,000, GTC_ERR_INVALID) with the
 * restrictions evaluated by sm_100a kernels, and builds the resident space of
 * the valid configurations in canonical order with coordinates rank/(k-1)
 * (GTC_ERR_EMPTY when nothing is valid). */
int gtc_space_enumerate(int device, const gtc_param_def* params, int32_t n_params,
                        const char* const* restrictions, int32_t n_restrictions,
                        int64_t* error_position, gtc_space** out);
/* Canonical indices (Configuration::index) of an enumerated space, ascending
 * (GTC_ERR_INVALID for spaces built from explicit coordinates). */
int gtc_space_ids(const gtc_space* space, uint64_t* ids);
/* Initial-sample snap (draw_initial_sample, sampling.hpp:98-117): for each
 * of the n points (n x d row-major, [0,1]^d) the position of the nearest
 * configuration (squared Euclidean distance accumulated in parameter order,
 * lowest position on ties), computed on the space's device. */
int gtc_space_nearest(const gtc_space* space, const double* points, int32_t n, int64_t* positions);
/* SearchSpace::cartesian_size() of an enumerated space (0 otherwise). */
uint64_t gtc_space_cartesian_size(const gtc_space* space);
/* Restriction::parse (restriction.hpp:479-486) without enumerating: 0 if the
 * text is a well-typed boolean restriction over `params`, else GTC_ERR_PARSE
 * with the position in *error_position. */
int gtc_restriction_validate(const gtc_param_def* params, int32_t n_params, const char* text,
                             int64_t* error_position);

/* ---- BO run: resident GP + predictions over the whole space ----------------- */
int gtc_run_create(gtc_space* space, const gtc_model_config* config, gtc_run** out);
/* Back to the freshly created state (no observations, nothing visited, no
 * group) under a new config with the same n_max, keeping the device
 * allocations: a worker that runs many BO runs reuses one run handle instead
 * of a create/destroy pair (cudaFree synchronises the whole device). */
int gtc_run_reset(gtc_run* run, const gtc_model_config* config);
/* Pool of idle runs per space: gtc_run_acquire returns a reset idle run of the
 * same n_max (else a new one); gtc_run_release waits for the run's stream and
 * returns it to the pool.  gtc_space_destroy destroys the pooled runs, so
 * sweeps of many runs allocate (and synchronise the device for) one run per
 * concurrent worker instead of one per run. */
int gtc_run_acquire(gtc_space* space, const gtc_model_config* config, gtc_run** out);
int gtc_run_release(gtc_run* run);
int gtc_run_destroy(gtc_run* run);

/* GpModel::fit over candidates at `positions` (the fit_current lambda,
 * strategies.hpp:298-307 -> gp.hpp:81-135) including jitter escalation, then
 * the full predictive pass over every candidate (refresh_predictions,
 * strategies.hpp:366-387).  n == 0 gives the prior. */
int gtc_fit(gtc_run* run, const int64_t* positions, const double* y_raw, int32_t n,
            gtc_fit_info* info);

/* Appends one valid observation (strategies.hpp:444-449): incremental
 * bordered-Cholesky row + one new row of V = L^-1 K* over all candidates, and
 * the refreshed posterior.  Equivalent to a refit; escalates jitter and
 * refactorises when the new pivot fails, exactly like gp.hpp:116-129. */
int gtc_append(gtc_run* run, int64_t position, double y_raw, gtc_fit_info* info);

/* Rolls the model back to its first n observations: GpModel::fit of that
 * prefix.  O(n) and asynchronous (info = NULL) while the factor is at the base
 * jitter (the factor is prefix-stable); after a jitter escalation the prefix
 * is refactorised from the base jitter, synchronously. */
int gtc_truncate(gtc_run* run, int32_t n, gtc_fit_info* info);

/* Visited bookkeeping (RunContext::evaluate, strategies.hpp:183-186). */
int gtc_mark_visited(gtc_run* run, int64_t position);
int gtc_unmark_visited(gtc_run* run, int64_t position);
int64_t gtc_unvisited_count(const gtc_run* run);

/* Fused mean-variance -> lambda -> EI/PI/LCB -> masked argmax for every AF in
 * af_mask in one pass over the candidates (strategies.hpp:404-436,
 * acquisition.hpp:12-83, portfolio.hpp:32-61). */
int gtc_select(gtc_run* run, const gtc_select_args* args, gtc_select_result* out);

/* One loop iteration after an evaluation (strategies.hpp:440-449 then
 * :401-436), with a single host synchronisation: marks `position` visited;
 * if `valid`, appends (position, y_raw) like gtc_append; then, if `args` is
 * non-null and candidates remain, runs gtc_select for the next suggestion.
 * `out` gets positions -1 when no selection ran. */
int gtc_observe(gtc_run* run, int64_t position, double y_raw, int32_t valid,
                const gtc_select_args* args, gtc_select_result* out, gtc_fit_info* info);

/* ---- resident BO loop (simulation mode) ---------------------------------- */
/* The objective of a simulation-mode run is a replay table (values[pos], NaN =
 * runtime-invalid; cache.hpp:246-257).  gtc_run_set_values copies it to the
 * device (n == gtc_space_size); gtc_run_steps then runs up to k iterations of
 * the BO loop (strategies.hpp:401-449: best_candidate, portfolio.hpp:32-61, for
 * bo-ei / bo-poi / bo-lcb; the portfolio below for bo-multi /
 * bo-advanced-multi) without host round trips: each
 * step selects (args: exactly one AF bit, no exclusions; f_best_raw = the
 * current best valid observation), evaluates the table, marks the pick
 * visited and, when valid, appends it (bordered row + predictive pass).
 * records[i] = the i-th step's pick, value, lambda and contextual-variance
 * fallback flag; *done = steps run (< k only when every candidate has been
 * visited).  Same results as the gtc_observe loop.  A failed bordered pivot
 * is refactorised with escalated jitter as in gtc_append.
 * GTC_STEPS_HOLD_N (benchmarking the steady state at a fixed n): every valid
 * step replaces the observation appended by the previous one at row n0 (the
 * model's size at the call) and un-marks its position, so every step runs at
 * exactly n0 + 1 observations; f_best_raw is then min(args->f_best_raw, y). */
typedef struct {
  int64_t position;
  double value;        /* NaN when invalid */
  double lambda;       /* exploration factor of the selection that picked it */
  int32_t valid;
  int32_t cv_fallback; /* 1: contextual variance undefined, constant used */
  int32_t by;          /* GTC_AF_* that produced the pick */
  int32_t pad;
} gtc_step_record;
/* Portfolio of a multi / advanced-multi run (PortfolioConfig, portfolio.hpp:65-71;
 * order ei, poi, lcb).  gtc_run_set_portfolio starts a fresh portfolio (NULL or
 * mode NONE: single AF); gtc_run_steps then runs Portfolio::suggest/record
 * (portfolio.hpp:130-309) on the device every step, args->af_mask ignored, and
 * keeps the portfolio state across calls.  Invalid results are recorded as the
 * median of the model's training values (= the run's valid observations). */
#define GTC_PORTFOLIO_NONE 0
#define GTC_PORTFOLIO_MULTI 1
#define GTC_PORTFOLIO_ADVANCED 2
typedef struct {
  int32_t mode;
  int32_t skip_threshold;
  double discount;
  double required_improvement;
} gtc_portfolio_config;
int gtc_run_set_portfolio(gtc_run* run, const gtc_portfolio_config* config);
/* The device portfolio of gtc_run_steps driven by an explicit script (the
 * reference's Portfolio unit scenarios, test_portfolio.cpp): kind 0 =
 * Portfolio::suggest on the given per-function argmax positions (ei, poi,
 * lcb), kind 1 = Portfolio::record(af, value).  out[i] = the suggestion
 * (position, by; -1 for records) and the state after op i.  initial_active
 * (NULL: all) restricts PortfolioConfig::order to a subset. */
typedef struct {
  int32_t kind;
  int32_t af;
  int64_t picks[3];
  double value;
} gtc_portfolio_op;
typedef struct {
  int64_t position;
  int32_t by;
  int32_t active[3];
  int32_t duplicates[3];
  int32_t above[3];
  int32_t below[3];
  int32_t pad;
  double dos[3];
} gtc_portfolio_state;
int gtc_portfolio_trace(int device, const gtc_portfolio_config* config, const int32_t* initial_active,
                        int32_t n_ops, const gtc_portfolio_op* ops, gtc_portfolio_state* out);
/* Programmatic dependent launch between the run's kernels (default on): the
 * next kernel is scheduled while the current one drains.  Turn it off for runs
 * that share a device with many concurrently driven runs (gtc_run_bo_batch
 * does), where early-scheduled waiting blocks would take SM slots from the
 * other runs' streams.  Results are identical either way. */
int gtc_run_set_pdl(gtc_run* run, int32_t enable);
#define GTC_STEPS_HOLD_N 1
#define GTC_STEPS_TIMING 2 /* record CUDA events around each step's phases */
int gtc_run_set_values(gtc_run* run, const double* values, int64_t n);
int gtc_run_steps(gtc_run* run, const gtc_select_args* args, int32_t k, int32_t flags,
                  gtc_step_record* records, int32_t* done, gtc_fit_info* info);
/* CUDA-event milliseconds of the last gtc_run_steps chunk's device work. */
double gtc_last_steps_ms(const gtc_run* run);
/* With GTC_STEPS_TIMING: mean CUDA-event ms per step of the last chunk's
 * phases: out3[0] selection + advance, [1] bordered append, [2] predictive pass. */
int gtc_last_steps_phase_ms(const gtc_run* run, double* out3);

/* Mean posterior variance over the unvisited candidates (the initial
 * contextual-variance normaliser, strategies.hpp:392-397; 0 when empty). */
int gtc_mean_variance(gtc_run* run, double* mean_variance, int64_t* count);

/* Copies the current standardized posterior mean / variance of every
 * candidate (GpPrediction.mean/.variance, gp.hpp:62-69) into host arrays of
 * length gtc_space_size().  Visited candidates carry values too. */
int gtc_read_predictions(gtc_run* run, double* mean, double* variance);

/* Device-side timing helpers for benchmarks, active only when the process
 * runs with GTC_PHASE_EVENTS=1 (events between the kernels would stop them
 * from launching early): CUDA-event milliseconds of the last gtc_append's
 * predictive-pass kernel (0 if none). */
double gtc_last_pass_ms(const gtc_run* run);
/* CUDA-event milliseconds of the last gtc_observe's device work (all of its
 * kernels, first launch to last, excluding the result readback). */
double gtc_last_step_ms(const gtc_run* run);
/* CUDA-event milliseconds of the last appending gtc_observe's phases:
 * out3[0] mark + bordered-row update, [1] predictive pass, [2] selection
 * (GTC_ERR_INVALID if the last observe did not append). */
int gtc_last_phase_ms(const gtc_run* run, double* out3);
/* Diagnostics: %globaltimer phase marks (ns) of the last bordered-row update
 * seen by gtc_observe: [0] start, [1] factor staged, [2] Gram row, [3] forward
 * solve, [4] pivot/row written, [5] c/e rows, [6] statistics + beta. */
int gtc_debug_append_marks(const gtc_run* run, uint64_t* marks7);
/* Diagnostics of libraries built with -DGTC_SEL_TRACE (GTC_ERR_INVALID
 * otherwise): %globaltimer marks (ns), 8 per row: rows < grid = the last
 * selection's blocks, row 2040 the loop-mode append, row 2041 the pass. */
int gtc_debug_select_trace(uint64_t* marks, int32_t rows);
/* Diagnostics: how full V rebuilds (fits, refits, gtc_gp_predict) run in this
 * process -- 4 (default) the kernel values first, then persistent 64-row
 * passes on the FP64 tensor cores (mma.sync) + the posterior pass (mode 2
 * when the pass's rows of L exceed shared memory, n > ~380); 2 the kernel
 * values first, then 32-row FMA passes; 3 the 32-row passes on mma.sync +
 * the posterior pass; 1 one tensor-core pass with shared-memory-resident V
 * blocks + the posterior pass; 0 the streaming 8-row passes that re-read the
 * V prefix from HBM.  All write bit-identical V and posterior.  Returns the
 * previous mode; a negative `mode` only queries. */
int gtc_debug_set_rebuild(int32_t mode);
/* Diagnostics: how full factorisations (GpModel::fit, refits) run in this
 * process -- 1 (default) right-looking with the packed factor in shared memory
 * (n up to ~230), 0 the left-looking bordered rows; both produce the same
 * factor bit for bit.  Returns the previous mode; negative only queries. */
int gtc_debug_set_factor(int32_t mode);
/* Diagnostics: bordered rows (since the run was created) whose
 * V-column pivot was below the exactness margin, so the exact forward
 * substitution ran (as of the last synchronising call). */
int64_t gtc_run_exact_rows(const gtc_run* run);
/* The CUDA stream the run launches on (as an opaque integer, for NCCL). */
uint64_t gtc_run_stream(const gtc_run* run);

/* ---- stand-alone GpModel over arbitrary points (gp.hpp:81-168) --------------- */
/* X: n x d row-major, y: n raw observations. */
int gtc_gp_fit(int device, const gtc_kernel* kernel, const double* X, const double* y_raw,
               int32_t n, int32_t d, double noise, double jitter, gtc_gp** out,
               gtc_fit_info* info);
/* Posterior at m points (Xstar m x d row-major), standardized scale. */
int gtc_gp_predict(gtc_gp* gp, const double* Xstar, int64_t m, double* mean, double* variance);
int gtc_gp_info(const gtc_gp* gp, gtc_fit_info* info);
int gtc_gp_destroy(gtc_gp* gp);

/* ---- acquisition over caller spans (best_candidate, portfolio.hpp:32-61) ----- */
/* means/stds: n candidates (CandidateScores spans); excluded: optional n bytes. */
int gtc_best_candidate(int device, int32_t af, const double* means, const double* stds, int64_t n,
                       double best_std, double lambda, const uint8_t* excluded,
                       int64_t* position_out, double* score_out);

/* Host view of a space: row-major n x d coords (as passed to gtc_space_create). */
const double* gtc_space_coords(const gtc_space* space);
int32_t gtc_space_dimension(const gtc_space* space);
int32_t gtc_space_device(const gtc_space* space);

/* ---- whole BO run (run_bo, strategies.hpp:261-457) on the resident surrogate ---- */
/* StrategyId order of the BO strategies (strategies.hpp:25-30) */
#define GTC_STRATEGY_BO_ADVANCED_MULTI 0
#define GTC_STRATEGY_BO_MULTI 1
#define GTC_STRATEGY_BO_EI 2
#define GTC_STRATEGY_BO_POI 3
#define GTC_STRATEGY_BO_LCB 4

/* StrategyConfig (strategies.hpp:79-122), BO fields.  lengthscale = NaN and
 * discount = NaN select the reference defaults (1.5 / 2.0; 0.65 / 0.75); other
 * out-of-range values fail like the reference ("kernel lengthscale must be
 * positive", GTC_ERR_INVALID; "discount factor must be in (0,1)", GTC_ERR_CONFIG). */
typedef struct {
  int32_t strategy;
  uint64_t seed;
  int64_t budget;
  int64_t n_init;
  int32_t invalid_consumes_budget;
  int32_t nu;
  double lengthscale;
  double output_variance;
  double noise;
  double jitter;
  int32_t exploration_mode;
  double exploration_constant;
  double discount;
  double required_improvement;
  int32_t skip_threshold;
  int64_t lhs_restarts;
} gtc_bo_config;

/* Objective (measurement.hpp:43): return 1 and *value for a valid
 * measurement, 0 for a runtime-invalid one, < 0 to abort the run. */
typedef int (*gtc_objective_fn)(void* ctx, int64_t position, uint64_t id, double* value);

typedef struct {
  int64_t position;
  uint64_t id;          /* EvaluationRecord::config_index */
  double value;         /* NaN when invalid */
  int32_t valid;
  double best_so_far;
} gtc_bo_record;

typedef struct {
  int64_t evaluations;
  int64_t budget_consumed;
  int64_t invalid_count;
  int64_t surrogate_size;
  int64_t n_records;
  int64_t n_lambdas;    /* BO iterations (inspect-hook calls) */
  int64_t best_position;
  double best_value;
  int32_t n_warnings;
} gtc_bo_summary;

/* ids: canonical index of every position (ascending).  records/lambdas are
 * caller arrays of `capacity` entries (>= budget + invalid evaluations). */
int gtc_run_bo(gtc_space* space, const uint64_t* ids, const gtc_bo_config* config,
               gtc_objective_fn objective, void* ctx, gtc_bo_record* records, double* lambdas,
               int64_t capacity, gtc_bo_summary* summary);
/* Same, objective = replay table (values[pos], NaN = runtime-invalid), the
 * simulation mode of cache.hpp:246-257. */
int gtc_run_bo_table(gtc_space* space, const uint64_t* ids, const gtc_bo_config* config,
                     const double* values, gtc_bo_record* records, double* lambdas,
                     int64_t capacity, gtc_bo_summary* summary);

/* run_experiment's worker pool (experiment.hpp:313-358) for replay tables:
 * n_runs independent BO runs over one resident space and one value table,
 * `threads` host threads (<= 0: hardware concurrency), each driving its runs
 * one after another on its own CUDA streams, so the device interleaves the
 * runs' kernels.  Run i uses configs[i] and writes records/lambdas at
 * i * capacity, summaries[i] and statuses[i] (a GTC_* code).  Returns GTC_OK
 * when every run succeeded, else the first failing run's status. */
int gtc_run_bo_batch(gtc_space* space, const uint64_t* ids, const gtc_bo_config* configs, int32_t n_runs,
                     const double* values, int32_t threads, gtc_bo_record* records, double* lambdas,
                     int64_t capacity, gtc_bo_summary* summaries, int32_t* statuses);

/* Observe groups: the member threads of a group each drive their own run
 * (gtc_run_set_group); a grouped gtc_observe waits until every member has
 * issued one (or left) and then all of them run in shared launches (one
 * bordered-append, one predictive-pass, one selection launch per AF mask, one
 * read-back) -- same results as the single-run path.  Every member thread
 * joins before its first grouped call and leaves when it is done.  Runs of a
 * group must share one space. */
int gtc_group_create(int device, gtc_group** out);
int gtc_group_destroy(gtc_group* group);
int gtc_group_join(gtc_group* group);
int gtc_group_leave(gtc_group* group);
int gtc_run_set_group(gtc_run* run, gtc_group* group);

/* MeasurementCache::checksum (cache.hpp:55-70): FNV-1a over (index, "%.17g"
 * value or invalid reason) of the entries in ascending index order; reasons:
 * 0 valid, 1 compile_error, 2 runtime_error, 3 restricted.  Host only. */
uint64_t gtc_cache_checksum(const uint64_t* ids, const double* values, const uint8_t* reasons, int64_t n);

/* ---- candidate-axis sharding (very large spaces over several GPUs) --------- */
/* Each rank holds a contiguous slice of the global candidate list in its own
 * gtc_space; the GP state is replicated (every rank applies the same
 * observations with explicit coordinates, so the factors stay identical).
 * Per iteration: gtc_shard_observe -> exchange (var_sum, var_count) -> sum in
 * rank order -> gtc_shard_select -> exchange gtc_shard_selection records ->
 * the same deterministic merge on every rank (portfolio.hpp:32-61 rule:
 * highest score, lowest position; NaN never wins except as first candidate). */
typedef struct {
  int64_t best_position[3];  /* best non-NaN score per AF slot (global), -1 if none */
  double best_score[3];
  int64_t first_eligible;    /* lowest eligible global position, -1 if none */
  uint32_t first_nan_mask;   /* bit af: that first candidate's score is NaN */
  int64_t n_candidates;
  double lambda;
  double mean_variance;
  double best_std;
  int32_t cv_fallback;
} gtc_shard_selection;

/* GpModel::fit from explicit training coordinates (X: n x d row-major). */
int gtc_fit_points(gtc_run* run, const double* X, const double* y_raw, int32_t n, gtc_fit_info* info);
/* This run's candidates are global positions [offset, offset + space size). */
int gtc_run_set_shard(gtc_run* run, int64_t offset);
/* Observation with explicit coordinates x_new (d); local_pos >= 0 only on the
 * rank whose slice holds it (marks it visited).  Returns this shard's total of
 * the refreshed posterior variance over its unvisited candidates. */
int gtc_shard_observe(gtc_run* run, const double* x_new, int64_t local_pos, double y_raw, int32_t valid,
                      double* var_sum, int64_t* var_count, gtc_fit_info* info);
/* Local fused selection using the GLOBAL variance total (args->excluded in
 * global positions). */
int gtc_shard_select(gtc_run* run, const gtc_select_args* args, double global_var_sum,
                     int64_t global_var_count, gtc_shard_selection* out);

/* ---- device-resident candidate-axis sharding (gtc_run_steps over shards) -- */
/* The whole iteration stays on the device: per step every shard runs its
 * selection over its slice, the shards all-gather one record each (the
 * best non-NaN score/position per acquisition function, the first eligible
 * position, the winners' coordinates and V columns), every shard merges them
 * with best_candidate's rule (portfolio.hpp:32-61) and appends the same
 * bordered row from the winner's V column, then runs its predictive pass and
 * all-gathers its fixed-point variance accumulators (the global lambda,
 * strategies.hpp:404-418, summed exactly: bit-identical to one device).  Both
 * exchanges are enqueued on the run's stream: no host round trip per
 * iteration.  Picks, lambdas and the factor are identical to the unsharded
 * gtc_run_steps on the same inputs. */
typedef struct gtc_comm gtc_comm;
#define GTC_NCCL_ID_BYTES 128
/* ncclGetUniqueId (libnccl.so.2 is opened at run time); rank 0 creates it and
 * the caller distributes the bytes (MPI, torch.distributed, a file...). */
int gtc_comm_nccl_id(uint8_t* id_out /* GTC_NCCL_ID_BYTES */);
/* ncclCommInitRank on `device`: one rank per process (or per host thread). */
int gtc_comm_create_nccl(const uint8_t* id, int32_t rank, int32_t nranks, int32_t device, gtc_comm** out);
/* Wraps a caller-owned ncclComm_t (passed as void*; not destroyed with the gtc_comm). */
int gtc_comm_wrap_nccl(void* nccl_comm, gtc_comm** out);
/* nranks in-process shards (out[0..nranks)), each driven by its own host
 * thread, on any devices: exchanges are peer copies ordered by CUDA events. */
int gtc_comm_create_local(int32_t nranks, gtc_comm** out);
int gtc_comm_destroy(gtc_comm* comm);
int32_t gtc_comm_rank(const gtc_comm* comm);
int32_t gtc_comm_size(const gtc_comm* comm);
/* This run (its space = global candidates [offset, offset + gtc_space_size))
 * becomes rank gtc_comm_rank(comm) of a sharded run over n_global candidates.
 * offset must be a multiple of 256 (the tile size: the variance totals are then
 * bit-identical to one device).  Every rank fits the same observations with
 * gtc_fit_points, marks its own visited positions (local indices), sets the
 * GLOBAL value table (gtc_run_set_values with n = n_global) and calls
 * gtc_run_steps with the same arguments; records carry global positions.
 * comm = NULL detaches. */
int gtc_run_attach_comm(gtc_run* run, gtc_comm* comm, int64_t offset, int64_t n_global);

/* Per-candidate acquisition values (acquisition_{ei,pi,lcb}, acquisition.hpp:25-42;
 * the LCB slot returns -lcb like best_candidate's score, portfolio.hpp:47). */
int gtc_acquisition_scores(int device, int32_t af, const double* means, const double* stds,
                           int64_t n, double best_std, double lambda, double* scores_out);

#ifdef __cplusplus
}
#endif

#endif /* GRIDTUNE_CUDA_H_ */
