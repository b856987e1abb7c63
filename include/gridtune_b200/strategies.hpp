// run_bo over the resident device surrogate (strategies.hpp:75-457 of the
// reference, BO strategies only).  Same control flow, RNG stream, budget
// accounting and portfolio semantics; the per-iteration surrogate pass
// (refit + predict-all + lambda + acquisition + argmax) is replaced by
//   gtc_append   (bordered Cholesky row + one V row over all candidates)
//   gtc_select   (mean variance -> lambda -> EI/PI/LCB -> masked argmax)
// so no O(N) work remains on the host inside the loop.
#pragma once

#include <array>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <limits>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "gridtune_b200/portfolio.hpp"
#include "gridtune_b200/sampling.hpp"

namespace gridtune_b200 {

enum class StrategyId { bo_advanced_multi, bo_multi, bo_ei, bo_poi, bo_lcb };

inline const char* to_string(StrategyId id) {
  switch (id) {
    case StrategyId::bo_advanced_multi: return "bo-advanced-multi";
    case StrategyId::bo_multi: return "bo-multi";
    case StrategyId::bo_ei: return "bo-ei";
    case StrategyId::bo_poi: return "bo-poi";
    case StrategyId::bo_lcb: return "bo-lcb";
  }
  return "?";
}

inline std::optional<StrategyId> strategy_from_string(const std::string& s) {
  for (StrategyId id : {StrategyId::bo_advanced_multi, StrategyId::bo_multi, StrategyId::bo_ei,
                        StrategyId::bo_poi, StrategyId::bo_lcb})
    if (s == to_string(id)) return id;
  return std::nullopt;
}

/// StrategyConfig (strategies.hpp:79-122), BO fields.
struct StrategyConfig {
  StrategyId id = StrategyId::bo_advanced_multi;
  std::uint64_t seed = 0;
  std::size_t budget = 220;
  std::size_t n_init = 20;
  bool invalid_consumes_budget = true;
  MaternNu nu = MaternNu::three_halves;
  std::optional<double> lengthscale;
  double output_variance = 1.0;
  double noise = 1e-10;
  double jitter = 1e-6;
  ExplorationConfig exploration;
  std::optional<double> discount;
  double required_improvement = 0.1;
  int skip_threshold = 5;
  std::size_t lhs_restarts = 50;
  std::function<void(std::size_t, std::size_t, std::size_t, double)> inspect;

  double effective_lengthscale() const {
    if (lengthscale) return *lengthscale;
    return exploration.mode == ExplorationConfig::Mode::contextual_variance ? 1.5 : 2.0;
  }
  double effective_discount(PortfolioMode mode) const {
    if (discount) return *discount;
    return mode == PortfolioMode::multi ? 0.65 : 0.75;
  }
};

struct EvaluationRecord {
  ConfigIndex config_index = 0;
  std::optional<double> value;
  InvalidReason reason = InvalidReason::runtime_error;
  double best_so_far = std::numeric_limits<double>::infinity();
};

struct TuningRun {
  std::vector<EvaluationRecord> records;
  std::size_t evaluations = 0;
  std::size_t budget_consumed = 0;
  std::size_t invalid_count = 0;
  double best_value = std::numeric_limits<double>::infinity();
  std::optional<Configuration> best_config;
  std::size_t surrogate_size = 0;
  std::vector<std::string> warnings;
  std::vector<double> lambdas;  // lambda of every BO iteration (inspect hook values)

  double best_at(std::size_t evaluation_count) const {
    if (records.empty() || evaluation_count == 0) return std::numeric_limits<double>::infinity();
    return records[std::min(evaluation_count, records.size()) - 1].best_so_far;
  }
};

namespace detail {

/// Visited flags, budget accounting, never-revisit (strategies.hpp:159-232).
class RunContext {
 public:
  RunContext(const EnumeratedSpace& space, const Objective& objective, const StrategyConfig& config)
      : space_(space), objective_(objective), config_(config), visited_(space.size(), false) {}

  TuningRun& run() { return run_; }
  std::size_t unvisited_count() const { return space_.size() - visited_count_; }
  bool visited(std::size_t pos) const { return visited_[pos]; }
  bool has_budget() const { return run_.budget_consumed < config_.budget; }
  bool exhausted() const { return !has_budget() || unvisited_count() == 0; }
  std::span<const double> valid_observations() const { return valid_; }

  Measurement evaluate(std::size_t pos) {
    if (visited_[pos]) throw Error("internal: configuration evaluated twice");
    visited_[pos] = true;
    ++visited_count_;
    if (on_visit) on_visit(pos);
    const Measurement m = objective_(space_.config(pos));
    ++run_.evaluations;
    EvaluationRecord rec;
    rec.config_index = space_.id(pos);
    if (m.is_valid()) {
      ++run_.budget_consumed;
      const double v = *m.value;
      rec.value = v;
      valid_.push_back(v);
      if (v < run_.best_value) {
        run_.best_value = v;
        run_.best_config = space_.config(pos);
      }
    } else {
      if (config_.invalid_consumes_budget) ++run_.budget_consumed;
      rec.reason = m.reason;
      ++run_.invalid_count;
    }
    rec.best_so_far = run_.best_value;
    run_.records.push_back(rec);
    return m;
  }

  std::function<void(std::size_t)> on_visit;  // mirrors the visited mask onto the device

 private:
  const EnumeratedSpace& space_;
  const Objective& objective_;
  const StrategyConfig& config_;
  std::vector<bool> visited_;
  std::vector<double> valid_;
  std::size_t visited_count_ = 0;
  TuningRun run_;
};

}  // namespace detail

/// One run's resident surrogate (gtc_run) as an argmax source: positions are
/// space positions, candidates are the unvisited configurations.
/// Observe group of the calling thread (gtc_run_bo_batch sets it for its
/// worker threads): runs created on the thread join it.
inline gtc_group*& thread_observe_group() {
  static thread_local gtc_group* g = nullptr;
  return g;
}
/// Whether the calling thread is currently a member of its observe group.
inline bool& thread_group_member() {
  static thread_local bool m = false;
  return m;
}

class DeviceSurrogate : public ArgmaxSource {
 public:
  DeviceSurrogate(const EnumeratedSpace& space, const MaternKernel& kernel, double noise, double jitter,
                  std::size_t n_max)
      : space_(space) {
    const gtc_model_config cfg{kernel.c(), noise, jitter, static_cast<std::int32_t>(n_max)};
    // run handles come from the space's pool of idle runs (gtc_run_acquire /
    // gtc_run_release): a sweep allocates device memory once per concurrent run
    gtc_run* r = nullptr;
    check(gtc_run_acquire(space.device_space(), &cfg, &r));
    run_.reset(r, [](gtc_run* p) { gtc_run_release(p); });
    if (gtc_group* g = thread_observe_group()) {
      check(gtc_run_set_group(run_.get(), g));
      // a batch worker's run shares the device with many concurrent runs
      check(gtc_run_set_pdl(run_.get(), 0));
    }
  }

  /// Membership of the run's observe group for the BO loop: a thread that
  /// starts a later run leaves the group during that run's initial design
  /// (host LHS, snap, first fit) so it does not hold up the other members'
  /// rounds.  (A worker joins at its start, so the first runs' initial designs
  /// all finish before the first round.)
  struct GroupMembership {
    gtc_group* g;
    explicit GroupMembership(gtc_group* group) : g(group) {
      if (g && !thread_group_member()) {
        gtc_group_join(g);
        thread_group_member() = true;
      }
    }
    ~GroupMembership() {
      if (g && thread_group_member()) {
        gtc_group_leave(g);
        thread_group_member() = false;
      }
    }
  };

  gtc_run* handle() const { return run_.get(); }

  gtc_fit_info fit(const std::vector<std::size_t>& positions, const std::vector<double>& y) {
    std::vector<std::int64_t> p(positions.begin(), positions.end());
    gtc_fit_info info{};
    check(gtc_fit(run_.get(), p.data(), y.data(), static_cast<std::int32_t>(y.size()), &info));
    info_ = info;
    return info;
  }
  gtc_fit_info append(std::size_t pos, double y) {
    gtc_fit_info info{};
    check(gtc_append(run_.get(), static_cast<std::int64_t>(pos), y, &info));
    info_ = info;
    return info;
  }
  void mark_visited(std::size_t pos) { check(gtc_mark_visited(run_.get(), static_cast<std::int64_t>(pos))); }
  double mean_variance() {
    double mv = 0.0;
    std::int64_t cnt = 0;
    check(gtc_mean_variance(run_.get(), &mv, &cnt));
    return mv;
  }
  double standardize(double y_raw) const { return (y_raw - info_.y_mean) / info_.y_std; }

  /// Per-iteration selection parameters (lambda inputs).
  gtc_select_args args{};
  gtc_select_result last{};

  /// Evaluation outcome -> device (mark visited, bordered append when valid)
  /// and, when `next` is given, the next iteration's selection in the same
  /// round trip (gtc_observe); the result is served to the next argmax().
  gtc_fit_info observe(std::size_t pos, std::optional<double> value, const gtc_select_args* next) {
    gtc_fit_info info{};
    check(gtc_observe(run_.get(), static_cast<std::int64_t>(pos), value.value_or(0.0), value ? 1 : 0, next,
                      &last, &info));
    if (value) info_ = info;
    prefetched_mask_ = next ? next->af_mask : 0u;
    return info;
  }

  std::array<std::int64_t, 3> argmax(std::uint32_t mask, const std::vector<std::int64_t>& excluded) override {
    if (prefetched_mask_ && excluded.empty() && (mask & ~prefetched_mask_) == 0) {
      prefetched_mask_ = 0;
      return {last.position[0], last.position[1], last.position[2]};
    }
    prefetched_mask_ = 0;
    gtc_select_args a = args;
    a.af_mask = mask;
    a.excluded = excluded.empty() ? nullptr : excluded.data();
    a.n_excluded = static_cast<std::int32_t>(excluded.size());
    check(gtc_select(run_.get(), &a, &last));
    return {last.position[0], last.position[1], last.position[2]};
  }
  /// Simulation mode: the objective's replay table on the device (gtc_run_set_values).
  void set_values(const double* values) { check(gtc_run_set_values(run_.get(), values, static_cast<std::int64_t>(space_.size()))); }

  void detach_group() { check(gtc_run_set_group(run_.get(), nullptr)); }
  void set_portfolio(const gtc_portfolio_config& c) { check(gtc_run_set_portfolio(run_.get(), &c)); }

  /// Up to k resident iterations of a single-AF loop (gtc_run_steps).
  std::vector<gtc_step_record> steps(const gtc_select_args& a, std::size_t k) {
    prefetched_mask_ = 0;
    std::vector<gtc_step_record> recs(std::max<std::size_t>(k, 1));
    std::int32_t done = 0;
    gtc_fit_info info{};
    check(gtc_run_steps(run_.get(), &a, static_cast<std::int32_t>(k), 0, recs.data(), &done, &info));
    recs.resize(static_cast<std::size_t>(done));
    if (done > 0) info_ = info;
    return recs;
  }

  std::uint64_t id_at(std::int64_t p) const override { return space_.id(static_cast<std::size_t>(p)); }
  std::int64_t position_of_id(std::uint64_t id) const override {
    const std::size_t p = space_.position_of(id);
    return p == EnumeratedSpace::npos ? -1 : static_cast<std::int64_t>(p);
  }
  std::size_t candidate_count() const override {
    return static_cast<std::size_t>(gtc_unvisited_count(run_.get()));
  }

 private:
  const EnumeratedSpace& space_;
  std::shared_ptr<gtc_run> run_;
  gtc_fit_info info_{};
  std::uint32_t prefetched_mask_ = 0;
};

inline bool is_bayesian(StrategyId) { return true; }

/// Whether run_bo may run single-AF simulation-mode loops on the device
/// (GTC_RESIDENT_LOOP=0 forces the per-iteration gtc_observe loop).
inline bool resident_loop_enabled() {
  const char* e = std::getenv("GTC_RESIDENT_LOOP");
  return !(e && e[0] == '0');
}

/// run_bo (strategies.hpp:261-457).
/// `table`: the objective's replay table (values[pos], NaN = invalid) when the
/// objective is one (simulation mode, cache.hpp:246-257); single-AF strategies
/// then run their loop resident on the device (gtc_run_steps), same results.
inline TuningRun run_bo(const EnumeratedSpace& space, const Objective& objective, const StrategyConfig& config,
                        const double* table = nullptr) {
  if (space.size() <= config.n_init)
    throw SamplingError("space has " + std::to_string(space.size()) +
                        " valid configurations; need more than n_init = " + std::to_string(config.n_init));
  if (config.budget <= config.n_init) throw ConfigError("budget must exceed the initial sample size");

  Rng rng(config.seed);
  detail::RunContext ctx(space, objective, config);
  const MaternKernel kernel(config.nu, config.effective_lengthscale(), config.output_variance);
  // the GP can hold at most `budget` valid observations (every valid one is charged)
  DeviceSurrogate gp(space, kernel, config.noise, config.jitter, std::max<std::size_t>(config.budget, 1));
  ctx.on_visit = [&gp](std::size_t pos) { gp.mark_visited(pos); };

  const Objective counted = [&ctx](const Configuration& c) { return ctx.evaluate(c.position); };
  const std::size_t max_init = config.invalid_consumes_budget ? config.budget : std::numeric_limits<std::size_t>::max();
  const InitialSample init = draw_initial_sample(space, counted, config.n_init, rng, max_init, config.lhs_restarts);

  std::vector<std::size_t> train_pos = init.positions;
  std::vector<double> train_val = init.observations;
  gp.fit(train_pos, train_val);  // fit_current(), strategies.hpp:298-309

  std::optional<Portfolio> portfolio;
  std::optional<AcquisitionId> single;
  switch (config.id) {
    case StrategyId::bo_ei: single = AcquisitionId::ei; break;
    case StrategyId::bo_poi: single = AcquisitionId::poi; break;
    case StrategyId::bo_lcb: single = AcquisitionId::lcb; break;
    default: {
      PortfolioConfig pc;
      pc.mode = config.id == StrategyId::bo_multi ? PortfolioMode::multi : PortfolioMode::advanced_multi;
      pc.skip_threshold = config.skip_threshold;
      pc.discount = config.effective_discount(pc.mode);
      pc.required_improvement = config.required_improvement;
      portfolio.emplace(pc);
    }
  }

  // contextual-variance normalisers, frozen after the initial sample (:390-397)
  ContextualVarianceState cv;
  cv.initial_sample_mean = init.mean_observation();
  cv.initial_mean_variance = gp.mean_variance();
  bool warned = false;
  ctx.on_visit = nullptr;  // inside the loop gtc_observe marks visited on the device

  auto select_args = [&]() {
    gtc_select_args a{};
    a.lambda_mode = static_cast<std::int32_t>(config.exploration.mode);
    a.lambda_constant = config.exploration.constant;
    a.cv_initial_sample_mean = cv.initial_sample_mean;
    a.cv_initial_mean_variance = cv.initial_mean_variance;
    a.f_best_raw = ctx.run().best_value;
    if (single) {
      a.af_mask = 1u << static_cast<int>(*single);
    } else {  // every active function: covers multi's fused pass and advanced's consulted one
      for (AcquisitionId af : portfolio->active()) a.af_mask |= 1u << static_cast<int>(af);
    }
    return a;
  };

  const bool resident = table && !config.inspect && resident_loop_enabled();
  if (resident) {
    gp.set_values(table);
    if (portfolio) {  // Portfolio::suggest/record run on the device (gtc_run_set_portfolio)
      const gtc_portfolio_config pc{config.id == StrategyId::bo_multi ? GTC_PORTFOLIO_MULTI : GTC_PORTFOLIO_ADVANCED,
                                    portfolio->config().skip_threshold, portfolio->config().discount,
                                    portfolio->config().required_improvement};
      gp.set_portfolio(pc);
    }
    // a resident run never takes part in observe rounds (gtc_run_bo_batch):
    // it runs on its own stream and must not hold up the group's members
    gp.detach_group();
    if (thread_observe_group() && thread_group_member()) {
      gtc_group_leave(thread_observe_group());
      thread_group_member() = false;
    }
  }
  const DeviceSurrogate::GroupMembership membership(resident ? nullptr : thread_observe_group());
  while (!ctx.exhausted()) {
    if (resident && !train_pos.empty()) {
      // as many iterations as the budget surely allows, without host round
      // trips; the host replays the evaluations (same table) for its records
      const std::size_t k = std::min(config.budget - ctx.run().budget_consumed, ctx.unvisited_count());
      const std::vector<gtc_step_record> recs = gp.steps(select_args(), k);
      if (recs.empty()) break;
      for (const gtc_step_record& r : recs) {
        if (r.cv_fallback && !warned) {
          ctx.run().warnings.push_back(
              "contextual variance unavailable (non-positive observations or zero initial variance); "
              "falling back to constant exploration factor " + std::to_string(config.exploration.constant));
          warned = true;
        }
        const Measurement m = ctx.evaluate(static_cast<std::size_t>(r.position));
        if (m.is_valid() != (r.valid != 0)) throw Error("internal: resident loop and objective disagree");
        if (m.is_valid()) {
          train_pos.push_back(static_cast<std::size_t>(r.position));
          train_val.push_back(*m.value);
        }
        ctx.run().lambdas.push_back(r.lambda);
      }
      continue;
    }
    gp.args = select_args();

    std::size_t pick;
    AcquisitionId by;
    if (single) {
      pick = static_cast<std::size_t>(gp.argmax(1u << static_cast<int>(*single), {})[static_cast<int>(*single)]);
      by = *single;
    } else {
      const Portfolio::Suggestion s = portfolio->suggest(gp);
      pick = s.position;
      by = s.by;
    }
    const double lambda = gp.last.lambda;
    if (gp.last.cv_fallback && !warned) {
      ctx.run().warnings.push_back(
          "contextual variance unavailable (non-positive observations or zero initial variance); "
          "falling back to constant exploration factor " + std::to_string(config.exploration.constant));
      warned = true;
    }
    const Measurement m = ctx.evaluate(pick);
    if (portfolio) portfolio->record(by, space.id(pick), m.value, ctx.valid_observations());
    if (m.is_valid()) {
      train_pos.push_back(pick);
      train_val.push_back(*m.value);
    }
    // refit == bordered append (strategies.hpp:444-449), fused with the next
    // iteration's selection (:401-436) into one device round trip
    const gtc_select_args next = select_args();
    gp.observe(pick, m.value, ctx.exhausted() ? nullptr : &next);
    ctx.run().lambdas.push_back(lambda);
    if (config.inspect) config.inspect(ctx.run().evaluations, ctx.valid_observations().size(), train_pos.size(), lambda);
  }
  ctx.run().surrogate_size = train_pos.size();
  return std::move(ctx.run());
}

inline TuningRun run_strategy(const EnumeratedSpace& space, const Objective& objective, const StrategyConfig& config) {
  return run_bo(space, objective, config);
}

}  // namespace gridtune_b200
