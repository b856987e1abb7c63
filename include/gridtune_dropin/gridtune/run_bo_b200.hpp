// run_bo with the reference's signature, executed by the B200 library
// (the INTEGRATION.md §3 binding as compilable code).
//
//   TuningRun run_bo_b200(const EnumeratedSpace&, const Objective&, const StrategyConfig&)
//     == gridtune::run_bo (strategies.hpp:261-457): same preconditions, initial
//        design, surrogate, exploration factor, acquisition / portfolio, budget
//        accounting, records and warnings; the surrogate stays resident on the
//        device and each iteration is one gtc_observe (bordered Cholesky row +
//        one new row of V + fused selection), the objective is called on the
//        caller's thread exactly once per evaluation like the reference's.
//
// Include after the reference's include/ is on the path (this header pulls in
// the reference's own strategies.hpp for the types).
#pragma once

#include <cmath>
#include <cstdint>
#include <exception>
#include <limits>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "gridtune/gp.hpp"  // the drop-in (b200::check)
#include "gridtune/strategies.hpp"
#include "gridtune_cuda.h"

namespace gridtune {

namespace b200 {

struct ObjectiveBridge {
  const EnumeratedSpace* space = nullptr;
  const Objective* objective = nullptr;
  std::vector<InvalidReason> reason;  // by position, for the records
  std::exception_ptr error;

  static int call(void* ctx, std::int64_t position, std::uint64_t /*id*/, double* value) {
    auto* b = static_cast<ObjectiveBridge*>(ctx);
    try {
      const Measurement m = (*b->objective)(b->space->configs[static_cast<std::size_t>(position)]);
      if (m.is_valid()) {
        *value = *m.value;
        return 1;
      }
      b->reason[static_cast<std::size_t>(position)] = m.reason;
      return 0;
    } catch (...) {
      b->error = std::current_exception();
      return -1;
    }
  }
};

}  // namespace b200

inline TuningRun run_bo_b200(const EnumeratedSpace& space, const Objective& objective, const StrategyConfig& config) {
  // preconditions of run_bo (strategies.hpp:263-271), checked before any device work
  if (!is_bayesian(config.id)) throw ConfigError("run_bo requires a BO strategy id");
  if (space.size() <= config.n_init)
    throw SamplingError("space has " + std::to_string(space.size()) +
                        " valid configurations; need more than n_init = " + std::to_string(config.n_init));
  if (config.budget <= config.n_init) throw ConfigError("budget must exceed the initial sample size");

  const std::size_t N = space.size(), d = space.dimension();
  // the resident space (a long-lived integration caches it next to the EnumeratedSpace)
  std::vector<double> flat(N * d);
  std::vector<std::uint64_t> ids(N);
  for (std::size_t p = 0; p < N; ++p) {
    for (std::size_t j = 0; j < d; ++j) flat[p * d + j] = space.coords[p][j];
    ids[p] = space.configs[p].index;
  }
  gtc_space* raw = nullptr;
  b200::check(gtc_space_create(b200::device(), flat.data(), static_cast<std::int64_t>(N),
                               static_cast<std::int32_t>(d), &raw));
  const std::unique_ptr<gtc_space, int (*)(gtc_space*)> dspace(raw, gtc_space_destroy);

  gtc_bo_config c{};
  c.strategy = static_cast<std::int32_t>(config.id);  // bo_* share the order of GTC_STRATEGY_*
  c.seed = config.seed;
  c.budget = static_cast<std::int64_t>(config.budget);
  c.n_init = static_cast<std::int64_t>(config.n_init);
  c.invalid_consumes_budget = config.invalid_consumes_budget ? 1 : 0;
  c.nu = static_cast<std::int32_t>(config.nu);
  c.lengthscale = config.lengthscale ? *config.lengthscale : std::numeric_limits<double>::quiet_NaN();
  c.output_variance = config.output_variance;
  c.noise = config.noise;
  c.jitter = config.jitter;
  c.exploration_mode = config.exploration.mode == ExplorationConfig::Mode::contextual_variance
                           ? GTC_LAMBDA_CONTEXTUAL_VARIANCE
                           : GTC_LAMBDA_CONSTANT;
  c.exploration_constant = config.exploration.constant;
  c.discount = config.discount ? *config.discount : std::numeric_limits<double>::quiet_NaN();
  c.required_improvement = config.required_improvement;
  c.skip_threshold = config.skip_threshold;
  c.lhs_restarts = static_cast<std::int64_t>(config.lhs_restarts);

  b200::ObjectiveBridge bridge;
  bridge.space = &space;
  bridge.objective = &objective;
  bridge.reason.assign(N, InvalidReason::runtime_error);
  // every evaluation is a distinct candidate: at most N records
  const std::int64_t cap = static_cast<std::int64_t>(N) + 1;
  std::vector<gtc_bo_record> recs(static_cast<std::size_t>(cap));
  std::vector<double> lambdas(static_cast<std::size_t>(cap));
  gtc_bo_summary sum{};
  const int rc = gtc_run_bo(dspace.get(), ids.data(), &c, &b200::ObjectiveBridge::call, &bridge, recs.data(),
                            lambdas.data(), cap, &sum);
  if (bridge.error) std::rethrow_exception(bridge.error);
  b200::check(rc);

  TuningRun run;
  run.evaluations = static_cast<std::size_t>(sum.evaluations);
  run.budget_consumed = static_cast<std::size_t>(sum.budget_consumed);
  run.invalid_count = static_cast<std::size_t>(sum.invalid_count);
  run.best_value = sum.best_value;
  if (sum.best_position >= 0) run.best_config = space.configs[static_cast<std::size_t>(sum.best_position)];
  run.surrogate_size = static_cast<std::size_t>(sum.surrogate_size);
  std::size_t valid_so_far = 0;
  std::vector<std::size_t> valid_after(static_cast<std::size_t>(sum.n_records));
  for (std::int64_t i = 0; i < sum.n_records; ++i) {
    const gtc_bo_record& r = recs[static_cast<std::size_t>(i)];
    EvaluationRecord e;
    e.config_index = r.id;
    if (r.valid) {
      e.value = r.value;
      ++valid_so_far;
    } else {
      e.reason = bridge.reason[static_cast<std::size_t>(r.position)];
    }
    e.best_so_far = r.best_so_far;
    run.records.push_back(e);
    valid_after[static_cast<std::size_t>(i)] = valid_so_far;
  }
  if (sum.n_warnings > 0)  // the one warning run_bo can emit (strategies.hpp:410-415)
    run.warnings.push_back(
        "contextual variance unavailable (non-positive observations or zero initial variance); falling back to "
        "constant exploration factor " +
        std::to_string(config.exploration.constant));
  if (config.inspect) {  // replayed per BO iteration: (evaluations, valid, GP size, lambda)
    const std::int64_t first = sum.n_records - sum.n_lambdas;
    for (std::int64_t k = 0; k < sum.n_lambdas; ++k) {
      const std::size_t r = static_cast<std::size_t>(first + k);
      config.inspect(r + 1, valid_after[r], valid_after[r], lambdas[static_cast<std::size_t>(k)]);
    }
  }
  return run;
}

}  // namespace gridtune
