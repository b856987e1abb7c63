// C ABI entry points for a whole BO run (gtc_run_bo / gtc_run_bo_table) over
// the C++ host mirror in include/gridtune_b200/strategies.hpp.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <exception>
#include <limits>
#include <string>

#include "gridtune_b200/strategies.hpp"

using namespace gridtune_b200;

// gtc_last_error() reads the kernel layer's message; host-layer exception
// text goes through the same thread-local channel (gtc_capi.cu).
extern "C" void gtc_internal_set_error(const char* msg);

namespace {

int to_status(const std::exception& e) {
  gtc_internal_set_error(e.what());
  if (dynamic_cast<const ModelConditioningError*>(&e)) return GTC_ERR_CONDITIONING;
  if (dynamic_cast<const ConfigError*>(&e)) return GTC_ERR_CONFIG;
  if (dynamic_cast<const SamplingError*>(&e)) return GTC_ERR_SAMPLING;
  if (dynamic_cast<const DeviceError*>(&e)) return GTC_ERR_CUDA;
  return GTC_ERR_INVALID;
}

StrategyConfig to_config(const gtc_bo_config& c) {
  if (c.strategy < 0 || c.strategy > 4) throw ConfigError("run_bo requires a BO strategy id");
  StrategyConfig s;
  s.id = static_cast<StrategyId>(c.strategy);
  s.seed = c.seed;
  s.budget = static_cast<std::size_t>(c.budget);
  s.n_init = static_cast<std::size_t>(c.n_init);
  s.invalid_consumes_budget = c.invalid_consumes_budget != 0;
  s.nu = static_cast<MaternNu>(c.nu);
  if (!std::isnan(c.lengthscale)) s.lengthscale = c.lengthscale;  // NaN: the reference default; <= 0 throws downstream
  s.output_variance = c.output_variance;
  s.noise = c.noise;
  s.jitter = c.jitter;
  s.exploration.mode = static_cast<ExplorationConfig::Mode>(c.exploration_mode);
  s.exploration.constant = c.exploration_constant;
  if (!std::isnan(c.discount)) s.discount = c.discount;  // NaN: the reference default; outside (0,1) throws downstream
  s.required_improvement = c.required_improvement;
  s.skip_threshold = c.skip_threshold;
  s.lhs_restarts = static_cast<std::size_t>(c.lhs_restarts);
  return s;
}

struct Aborted : std::exception {
  const char* what() const noexcept override { return "objective aborted the run"; }
};

int run(gtc_space* space, const std::uint64_t* ids, const gtc_bo_config* cfg, const Objective& objective,
        gtc_bo_record* records, double* lambdas, std::int64_t capacity, gtc_bo_summary* summary,
        const double* table = nullptr) {
  if (!space || !ids || !cfg) {
    gtc_internal_set_error("null argument");
    return GTC_ERR_INVALID;
  }
  try {
    const EnumeratedSpace es(space, ids);
    const StrategyConfig sc = to_config(*cfg);
    const TuningRun r = run_bo(es, objective, sc, table);
    const std::int64_t nrec = static_cast<std::int64_t>(r.records.size());
    const std::int64_t nlam = static_cast<std::int64_t>(r.lambdas.size());
    if (records) {
      if (nrec > capacity) throw Error("record capacity too small");
      for (std::int64_t i = 0; i < nrec; ++i) {
        const EvaluationRecord& e = r.records[static_cast<std::size_t>(i)];
        records[i].id = e.config_index;
        records[i].position = static_cast<std::int64_t>(es.position_of(e.config_index));
        records[i].valid = e.value.has_value() ? 1 : 0;
        records[i].value = e.value ? *e.value : std::numeric_limits<double>::quiet_NaN();
        records[i].best_so_far = e.best_so_far;
      }
    }
    if (lambdas) {
      if (nlam > capacity) throw Error("lambda capacity too small");
      for (std::int64_t i = 0; i < nlam; ++i) lambdas[i] = r.lambdas[static_cast<std::size_t>(i)];
    }
    if (summary) {
      summary->evaluations = static_cast<std::int64_t>(r.evaluations);
      summary->budget_consumed = static_cast<std::int64_t>(r.budget_consumed);
      summary->invalid_count = static_cast<std::int64_t>(r.invalid_count);
      summary->surrogate_size = static_cast<std::int64_t>(r.surrogate_size);
      summary->n_records = nrec;
      summary->n_lambdas = nlam;
      summary->best_value = r.best_value;
      summary->best_position = r.best_config ? static_cast<std::int64_t>(r.best_config->position) : -1;
      summary->n_warnings = static_cast<std::int32_t>(r.warnings.size());
    }
    return GTC_OK;
  } catch (const Aborted& e) {
    gtc_internal_set_error(e.what());
    return GTC_ERR_ABORTED;
  } catch (const std::exception& e) {
    return to_status(e);
  }
}

}  // namespace

extern "C" int gtc_run_bo(gtc_space* space, const std::uint64_t* ids, const gtc_bo_config* cfg,
                          gtc_objective_fn objective, void* ctx, gtc_bo_record* records, double* lambdas,
                          std::int64_t capacity, gtc_bo_summary* summary) {
  if (!objective) {
    gtc_internal_set_error("objective is null");
    return GTC_ERR_INVALID;
  }
  const Objective obj = [objective, ctx](const Configuration& c) {
    double v = 0.0;
    const int rc = objective(ctx, static_cast<std::int64_t>(c.position), c.index, &v);
    if (rc < 0) throw Aborted();
    return rc > 0 ? Measurement::valid(v) : Measurement::invalid(InvalidReason::runtime_error);
  };
  return run(space, ids, cfg, obj, records, lambdas, capacity, summary);
}

extern "C" int gtc_run_bo_batch(gtc_space* space, const std::uint64_t* ids, const gtc_bo_config* configs,
                                std::int32_t n_runs, const double* values, std::int32_t threads,
                                gtc_bo_record* records, double* lambdas, std::int64_t capacity,
                                gtc_bo_summary* summaries, std::int32_t* statuses) {
  if (!space || !ids || !configs || !values || !statuses || n_runs < 0) {
    gtc_internal_set_error("null argument");
    return GTC_ERR_INVALID;
  }
  const Objective obj = [values](const Configuration& c) {
    const double v = values[c.position];
    return std::isnan(v) ? Measurement::invalid(InvalidReason::runtime_error) : Measurement::valid(v);
  };
  int workers = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  workers = std::max(1, std::min(workers, static_cast<int>(n_runs)));
  // observe groups: each group's per-iteration device work shares launches;
  // several groups (own streams) keep the device busy while one group's
  // threads do their host work
  static const int per_group = [] {
    const char* e = std::getenv("GTC_RUNS_PER_GROUP");
    return e ? std::max(1, std::atoi(e)) : 64;
  }();
  const int n_groups = workers > 1 ? (workers + per_group - 1) / per_group : 0;
  std::vector<gtc_group*> groups(n_groups, nullptr);
  for (int k = 0; k < n_groups; ++k) {
    const int rc = gtc_group_create(gtc_space_device(space), &groups[k]);
    if (rc) {
      for (gtc_group* g : groups) gtc_group_destroy(g);
      return rc;
    }
  }
  // GTC_BATCH_RESIDENT=1: single-AF runs loop resident on the device
  // (gtc_run_steps, own stream) instead of joining the observe groups
  const char* br = std::getenv("GTC_BATCH_RESIDENT");
  const bool batch_resident = br && br[0] == '1';
  std::atomic<std::int32_t> next{0}, next_worker{0};
  auto worker = [&]() {
    const int w = next_worker.fetch_add(1);
    // the worker is a member from its start until its first run's loop ends;
    // later runs join for their BO loops only (run_bo's GroupMembership)
    gtc_group* group = n_groups ? groups[w % n_groups] : nullptr;
    thread_observe_group() = group;
    if (group) {
      gtc_group_join(group);
      thread_group_member() = true;
    }
    for (std::int32_t i; (i = next.fetch_add(1)) < n_runs;) {
      statuses[i] = run(space, ids, &configs[i], obj, records ? records + (std::int64_t)i * capacity : nullptr,
                        lambdas ? lambdas + (std::int64_t)i * capacity : nullptr, capacity,
                        summaries ? &summaries[i] : nullptr, batch_resident ? values : nullptr);
    }
    if (group && thread_group_member()) gtc_group_leave(group);  // (a run that failed early)
    thread_group_member() = false;
    thread_observe_group() = nullptr;
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < workers; ++w) pool.emplace_back(worker);
  worker();
  for (std::thread& t : pool) t.join();
  for (gtc_group* g : groups) gtc_group_destroy(g);
  for (std::int32_t i = 0; i < n_runs; ++i)
    if (statuses[i] != GTC_OK) return statuses[i];
  return GTC_OK;
}

extern "C" int gtc_run_bo_table(gtc_space* space, const std::uint64_t* ids, const gtc_bo_config* cfg,
                                const double* values, gtc_bo_record* records, double* lambdas,
                                std::int64_t capacity, gtc_bo_summary* summary) {
  if (!values) {
    gtc_internal_set_error("values is null");
    return GTC_ERR_INVALID;
  }
  const Objective obj = [values](const Configuration& c) {
    const double v = values[c.position];
    return std::isnan(v) ? Measurement::invalid(InvalidReason::runtime_error) : Measurement::valid(v);
  };
  return run(space, ids, cfg, obj, records, lambdas, capacity, summary, values);
}
