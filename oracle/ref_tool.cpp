// ref_tool — TEST INFRASTRUCTURE ONLY.  Drives the UNMODIFIED reference
// (/root/reference/proj/include/gridtune, header-only) compiled against the
// in-repo Eigen/GTest shims (oracle/shim) to
//   * produce golden vectors for tests/golden (scripted by tests/golden/make_golden.py),
//   * produce reference run_bo trajectories for the trajectory parity tests,
//   * time the reference CPU path for bench.py --impl reference / cpu_baseline.
// Nothing in the product links this file.  Output: .npy files + JSON on stdout.
//
// Usage:
//   ref_tool space  <function> <grid AxBx..> <seed> <invalid|-> <outdir>
//   ref_tool gemm   <outdir>                      # C1 GEMM space (restriction parser)
//   ref_tool gp     <seed> <trials> <outdir>      # GpModel fit/predict golden vectors
//   ref_tool runbo  <function> <grid> <seed> <invalid|-> <strategy> <budget> <n_init> <bo_seed> <outdir>
//   ref_tool bench  <grid> <seed> <n> <threads> <steps> <af>   # CPU baseline (JSON line)
//   ref_tool enumjson <spec.json> <outdir>        # SearchSpace(params, restrictions) + EnumeratedSpace
//   ref_tool restrict <spec.json>                 # Restriction::parse + evaluate over the grid
//   ref_tool cachegen <function> <grid> <seed> <invalid|-> <path>   # MeasurementCache::save (JSON)
//   ref_tool runbo_spec <spec.json> <values.f64> <strategy> <budget> <n_init> <bo_seed> <outdir>
#include <chrono>
#include <cmath>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "gridtune/experiment.hpp"
#include "gridtune/strategies.hpp"
#include "gridtune/synthetic.hpp"
#include "json.hpp"

using namespace gridtune;
namespace fs = std::filesystem;

namespace {

// ---- minimal .npy writer (little-endian, C order) ----
template <class T>
const char* npy_descr();
template <>
const char* npy_descr<double>() { return "<f8"; }
template <>
const char* npy_descr<std::int64_t>() { return "<i8"; }
template <>
const char* npy_descr<std::uint64_t>() { return "<u8"; }
template <>
const char* npy_descr<std::uint8_t>() { return "|u1"; }

template <class T>
void write_npy(const fs::path& path, const std::vector<T>& data, std::vector<std::size_t> shape) {
  std::ostringstream h;
  h << "{'descr': '" << npy_descr<T>() << "', 'fortran_order': False, 'shape': (";
  for (std::size_t i = 0; i < shape.size(); ++i) h << shape[i] << (shape.size() == 1 ? "," : (i + 1 < shape.size() ? ", " : ""));
  h << "), }";
  std::string header = h.str();
  const std::size_t total = 10 + header.size() + 1;
  header += std::string((64 - total % 64) % 64, ' ') + "\n";
  std::ofstream f(path, std::ios::binary);
  f.write("\x93NUMPY\x01\x00", 8);
  const std::uint16_t hl = static_cast<std::uint16_t>(header.size());
  f.write(reinterpret_cast<const char*>(&hl), 2);
  f.write(header.data(), static_cast<std::streamsize>(header.size()));
  f.write(reinterpret_cast<const char*>(data.data()), static_cast<std::streamsize>(sizeof(T) * data.size()));
}

std::vector<std::size_t> parse_grid(const std::string& s) {
  std::vector<std::size_t> g;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, 'x')) g.push_back(std::stoul(tok));
  return g;
}

MeasurementCache make_cache(const std::string& fn, const std::string& grid, std::uint64_t seed,
                            const std::string& invalid) {
  SyntheticSpec spec;
  spec.function = fn;
  spec.grid = parse_grid(grid);
  spec.seed = seed;
  if (invalid != "-") spec.invalid_fraction = std::stod(invalid);
  return generate_synthetic(spec);
}

void dump_space(const EnumeratedSpace& space, const MeasurementCache* cache, const fs::path& out) {
  fs::create_directories(out);
  const std::size_t N = space.size(), d = space.dimension();
  std::vector<double> coords(N * d), values(N);
  std::vector<std::uint64_t> ids(N);
  for (std::size_t p = 0; p < N; ++p) {
    for (std::size_t j = 0; j < d; ++j) coords[p * d + j] = space.coords[p][j];
    ids[p] = space.configs[p].index;
    values[p] = std::numeric_limits<double>::quiet_NaN();
    if (cache) {
      const Measurement& m = cache->entries.at(space.configs[p].index);
      if (m.is_valid()) values[p] = *m.value;
    }
  }
  write_npy(out / "coords.npy", coords, {N, d});
  write_npy(out / "ids.npy", ids, {N});
  if (cache) write_npy(out / "values.npy", values, {N});
}

StrategyId strategy_of(const std::string& s) {
  auto id = strategy_from_string(s);
  if (!id) throw ConfigError("unknown strategy " + s);
  return *id;
}

int cmd_space(int argc, char** argv) {
  if (argc < 7) return 2;
  const MeasurementCache cache = make_cache(argv[2], argv[3], std::stoull(argv[4]), argv[5]);
  const EnumeratedSpace space(cache.space());
  dump_space(space, &cache, argv[6]);
  std::printf("{\"n\": %zu, \"d\": %zu, \"invalid\": %zu, \"true_minimum\": %.17g}\n", space.size(),
              space.dimension(), cache.invalid_count(), *cache.true_minimum);
  return 0;
}

// C1: the GEMM search space of PAPER.md:319-333 with Kernel Tuner's
// restrictions, enumerated by the reference's own parser.
int cmd_gemm(int argc, char** argv) {
  if (argc < 3) return 2;
  std::vector<ParameterDef> p{
      ParameterDef("MWG", {16, 32, 64, 128}), ParameterDef("NWG", {16, 32, 64, 128}),
      ParameterDef("KWG", {32}),              ParameterDef("MDIMC", {8, 16, 32}),
      ParameterDef("NDIMC", {8, 16, 32}),     ParameterDef("MDIMA", {8, 16, 32}),
      ParameterDef("NDIMB", {8, 16, 32}),     ParameterDef("KWI", {2}),
      ParameterDef("VWM", {1, 2, 4, 8}),      ParameterDef("VWN", {1, 2, 4, 8}),
      ParameterDef("STRM", {0}),              ParameterDef("STRN", {0}),
      ParameterDef("SA", {0, 1}),             ParameterDef("SB", {0, 1}),
      ParameterDef("PRECISION", {32})};
  const std::vector<std::string> r{"KWG % KWI == 0",
                                   "MWG % (MDIMC * VWM) == 0",
                                   "NWG % (NDIMC * VWN) == 0",
                                   "MWG % (MDIMA * VWM) == 0",
                                   "NWG % (NDIMB * VWN) == 0",
                                   "KWG % ((MDIMC * NDIMC) / MDIMA) == 0",
                                   "KWG % ((MDIMC * NDIMC) / NDIMB) == 0"};
  const SearchSpace s(p, r);
  const EnumeratedSpace space(s);
  dump_space(space, nullptr, argv[2]);
  std::printf("{\"n\": %zu, \"d\": %zu, \"cartesian\": %" PRIu64 "}\n", space.size(), space.dimension(),
              s.cartesian_size());
  return 0;
}

// GpModel golden vectors in the style of test_gp.cpp:87-126.
int cmd_gp(int argc, char** argv) {
  if (argc < 5) return 2;
  Rng rng(std::stoull(argv[2]));
  const int trials = std::stoi(argv[3]);
  const fs::path out = argv[4];
  fs::create_directories(out);
  for (int t = 0; t < trials; ++t) {
    const std::size_t n = 1 + rng.uniform_below(40);
    const std::size_t d = 1 + rng.uniform_below(6);
    const MaternNu nu = static_cast<MaternNu>(t % 3);
    const double l = 0.3 + 2.5 * rng.uniform01();
    const double s2 = 0.5 + rng.uniform01();
    const MaternKernel kernel(nu, l, s2);
    Eigen::MatrixXd X(n, d), Q(64, d);
    Eigen::VectorXd y(n);
    for (std::size_t i = 0; i < n; ++i) {
      for (std::size_t j = 0; j < d; ++j) X(i, j) = rng.uniform01();
      y(i) = 5.0 + 3.0 * rng.normal();
    }
    for (int i = 0; i < 64; ++i)
      for (std::size_t j = 0; j < d; ++j) Q(i, j) = rng.uniform01();
    const GpModel model = GpModel::fit(kernel, X, y);
    const GpPrediction p = model.predict(Q);
    std::vector<double> Xv(n * d), Qv(64 * d), yv(n), mv(64), vv(64);
    for (std::size_t i = 0; i < n; ++i) {
      yv[i] = y(i);
      for (std::size_t j = 0; j < d; ++j) Xv[i * d + j] = X(i, j);
    }
    for (int i = 0; i < 64; ++i) {
      mv[i] = p.mean(i);
      vv[i] = p.variance(i);
      for (std::size_t j = 0; j < d; ++j) Qv[i * d + j] = Q(i, j);
    }
    const std::string pre = "gp" + std::to_string(t) + "_";
    write_npy(out / (pre + "X.npy"), Xv, {n, d});
    write_npy(out / (pre + "y.npy"), yv, {n});
    write_npy(out / (pre + "Q.npy"), Qv, {64, d});
    write_npy(out / (pre + "mean.npy"), mv, {64});
    write_npy(out / (pre + "var.npy"), vv, {64});
    write_npy(out / (pre + "meta.npy"),
              std::vector<double>{static_cast<double>(nu), l, s2, model.y_mean(), model.y_std(), model.jitter()},
              {6});
  }
  std::printf("{\"trials\": %d}\n", trials);
  return 0;
}

int cmd_runbo(int argc, char** argv) {
  if (argc < 11) return 2;
  const MeasurementCache cache = make_cache(argv[2], argv[3], std::stoull(argv[4]), argv[5]);
  const EnumeratedSpace space(cache.space());
  StrategyConfig config;
  config.id = strategy_of(argv[6]);
  config.budget = std::stoul(argv[7]);
  config.n_init = std::stoul(argv[8]);
  config.seed = std::stoull(argv[9]);
  const fs::path out = argv[10];
  std::vector<double> lambdas;
  config.inspect = [&](std::size_t, std::size_t, std::size_t, double l) { lambdas.push_back(l); };
  const TuningRun run = run_bo(space, cache.objective(), config);
  dump_space(space, &cache, out);
  std::vector<std::int64_t> pos;
  std::vector<double> val;
  for (const EvaluationRecord& r : run.records) {
    pos.push_back(static_cast<std::int64_t>(space.position_of(r.config_index)));
    val.push_back(r.value ? *r.value : std::numeric_limits<double>::quiet_NaN());
  }
  write_npy(out / "traj_pos.npy", pos, {pos.size()});
  write_npy(out / "traj_val.npy", val, {val.size()});
  write_npy(out / "traj_lambda.npy", lambdas, {lambdas.size()});
  std::printf("{\"evaluations\": %zu, \"best\": %.17g, \"surrogate\": %zu, \"warnings\": %zu}\n",
              run.evaluations, run.best_value, run.surrogate_size, run.warnings.size());
  return 0;
}

// Reference CPU path for one BO iteration at (N, n): GpModel::fit over the n
// observations + GpModel::predict over every unvisited candidate (split over
// `threads` host threads, each calling the reference's predict on its slice)
// + mean variance + contextual lambda + best_candidate (strategies.hpp:366-436).
int cmd_bench(int argc, char** argv) {
  if (argc < 8) return 2;
  // optional argv[8]: the workload's runtime-invalid fraction (C3: 0.3)
  const MeasurementCache cache = make_cache("random-rough", argv[2], std::stoull(argv[3]), argc > 8 ? argv[8] : "0");
  const EnumeratedSpace space(cache.space());
  const std::size_t n = std::stoul(argv[4]);
  const unsigned threads = std::max(1u, static_cast<unsigned>(std::stoul(argv[5])));
  const int steps = std::stoi(argv[6]);
  const std::string af_name = argv[7];
  if (af_name != "ei" && af_name != "poi" && af_name != "lcb") {
    std::fprintf(stderr, "unknown acquisition function '%s' (ei, poi, lcb)\n", af_name.c_str());
    return 2;
  }
  const AcquisitionId af = af_name == "ei" ? AcquisitionId::ei : af_name == "poi" ? AcquisitionId::poi : AcquisitionId::lcb;
  const std::size_t N = space.size(), d = space.dimension();
  const Objective objective = cache.objective();
  Rng rng(12345);
  std::vector<bool> visited(N, false);
  std::vector<std::size_t> train;
  std::vector<double> vals;
  while (train.size() < n) {
    const std::size_t p = rng.uniform_below(N);
    if (visited[p]) continue;
    const auto m = objective(space.configs[p]);
    if (!m.value) continue;  // runtime-invalid: never reaches the GP (strategies.hpp:444-449)
    visited[p] = true;
    train.push_back(p);
    vals.push_back(*m.value);
  }
  Eigen::MatrixXd X(n, d);
  Eigen::VectorXd y(n);
  for (std::size_t i = 0; i < n; ++i) {
    for (std::size_t j = 0; j < d; ++j) X(i, j) = space.coords[train[i]][j];
    y(i) = vals[i];
  }
  std::vector<std::size_t> cand;
  for (std::size_t p = 0; p < N; ++p)
    if (!visited[p]) cand.push_back(p);
  const std::size_t U = cand.size();
  const MaternKernel kernel(MaternNu::three_halves, 1.5, 1.0);
  double total = 0.0;
  std::size_t last_pick = 0;
  for (int step = 0; step < steps; ++step) {
    const auto t0 = std::chrono::steady_clock::now();
    const GpModel model = GpModel::fit(kernel, X, y, 1e-10, 1e-6);
    std::vector<double> means(U), stds(U), vars(U);
    std::vector<std::thread> pool;
    const std::size_t chunk = (U + threads - 1) / threads;
    for (unsigned t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        const std::size_t lo0 = t * chunk, hi0 = std::min(U, lo0 + chunk);
        // sub-chunks bound the eager temporaries (n x chunk) per call; predict
        // is column-independent so results equal one big call
        constexpr std::size_t kSub = 16384;
        for (std::size_t lo = lo0; lo < hi0; lo += kSub) {
          const std::size_t hi = std::min(hi0, lo + kSub);
          Eigen::MatrixXd Xs(hi - lo, d);
          for (std::size_t i = lo; i < hi; ++i)
            for (std::size_t j = 0; j < d; ++j) Xs(i - lo, j) = space.coords[cand[i]][j];
          const GpPrediction p = model.predict(Xs);
          for (std::size_t i = lo; i < hi; ++i) {
            means[i] = p.mean(i - lo);
            vars[i] = p.variance(i - lo);
            stds[i] = std::sqrt(vars[i]);
          }
        }
      });
    }
    for (auto& th : pool) th.join();
    double best = vals[0];
    for (double v : vals) best = std::min(best, v);
    const double mean_var = std::accumulate(vars.begin(), vars.end(), 0.0) / static_cast<double>(U);
    ContextualVarianceState cv{std::accumulate(vals.begin(), vals.begin() + std::min<std::size_t>(20, n), 0.0) /
                                   static_cast<double>(std::min<std::size_t>(20, n)),
                               mean_var};
    const double lambda = contextual_variance_lambda(cv, mean_var, best).value_or(0.01);
    std::vector<std::uint64_t> ids(U);
    for (std::size_t i = 0; i < U; ++i) ids[i] = space.configs[cand[i]].index;
    CandidateScores scores{ids, means, stds, model.standardize(best), lambda};
    last_pick = cand[best_candidate(af, scores)];
    total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  std::printf("{\"N\": %zu, \"n\": %zu, \"d\": %zu, \"threads\": %u, \"steps\": %d, \"seconds_per_step\": %.6f, "
              "\"iters_per_sec\": %.6g, \"last_pick\": %zu}\n",
              N, n, d, threads, steps, total / steps, steps / total, last_pick);
  return 0;
}

}  // namespace

// ---- search spaces from a JSON spec:
// {"params": [{"name": .., "kind": "numeric|categorical|boolean", "values": [..]}],
//  "restrictions": ["..", ..]}
std::vector<ParameterDef> params_from_json(const nlohmann::json& j) {
  std::vector<ParameterDef> ps;
  for (const auto& p : j.at("params")) {
    const std::string kind = p.at("kind");
    std::vector<Value> vals;
    for (const auto& v : p.at("values")) {
      if (kind == "numeric") vals.emplace_back(v.get<double>());
      else if (kind == "categorical") vals.emplace_back(v.get<std::string>());
      else vals.emplace_back(v.get<bool>());
    }
    ParameterDef d;  // unvalidated: SearchSpace validates (so its errors are reproduced)
    d.name = p.at("name");
    d.kind = kind == "numeric" ? ParamKind::numeric : kind == "categorical" ? ParamKind::categorical : ParamKind::boolean;
    d.values = std::move(vals);
    ps.push_back(std::move(d));
  }
  return ps;
}

std::string json_escape(const std::string& s) { return nlohmann::json(s).dump(); }

int cmd_enumjson(int argc, char** argv) {
  if (argc < 4) return 2;
  std::ifstream f(argv[2]);
  const nlohmann::json spec = nlohmann::json::parse(f);
  std::vector<std::string> rs = spec.value("restrictions", std::vector<std::string>{});
  try {
    SearchSpace s(params_from_json(spec), rs);
    const EnumeratedSpace space(s);
    dump_space(space, nullptr, argv[3]);
    std::printf("{\"n\": %zu, \"d\": %zu, \"cartesian\": %" PRIu64 "}\n", space.size(), space.dimension(),
                s.cartesian_size());
  } catch (const ParseError& e) {
    std::printf("{\"error\": \"parse\", \"message\": %s, \"position\": %zu}\n", json_escape(e.what()).c_str(),
                e.position());
  } catch (const EmptySearchSpaceError& e) {
    std::printf("{\"error\": \"empty\", \"message\": %s}\n", json_escape(e.what()).c_str());
  } catch (const Error& e) {
    std::printf("{\"error\": \"error\", \"message\": %s}\n", json_escape(e.what()).c_str());
  }
  return 0;
}

// One JSON line per restriction: the parse outcome, and for well-formed ones
// the truth value at every grid point (canonical order) as a 0/1 string.
int cmd_restrict(int argc, char** argv) {
  if (argc < 3) return 2;
  std::ifstream f(argv[2]);
  const nlohmann::json spec = nlohmann::json::parse(f);
  const std::vector<ParameterDef> ps = params_from_json(spec);
  const SearchSpace grid(ps);
  for (const std::string& text : spec.at("restrictions")) {
    try {
      const Restriction r = parse_restriction(text, ps);
      std::string bits;
      for (ConfigIndex i = 0; i < grid.cartesian_size(); ++i) bits += r.evaluate(grid.config_at(i).values) ? '1' : '0';
      std::printf("{\"text\": %s, \"ok\": true, \"bits\": \"%s\"}\n", json_escape(text).c_str(), bits.c_str());
    } catch (const ParseError& e) {
      std::printf("{\"text\": %s, \"ok\": false, \"message\": %s, \"position\": %zu}\n", json_escape(text).c_str(),
                  json_escape(e.what()).c_str(), e.position());
    }
  }
  return 0;
}

// run_bo of the reference over a JSON-specified space (SearchSpace +
// EnumeratedSpace) with replay values from a raw little-endian f64 file in
// position order (NaN = runtime-invalid): the simulation-mode C1/C2 cases.
int cmd_runbo_spec(int argc, char** argv) {
  if (argc < 9) return 2;
  std::ifstream f(argv[2]);
  const nlohmann::json spec = nlohmann::json::parse(f);
  std::vector<std::string> rs = spec.value("restrictions", std::vector<std::string>{});
  const SearchSpace ss(params_from_json(spec), rs);
  const EnumeratedSpace space(ss);
  std::vector<double> values(space.size());
  std::ifstream vf(argv[3], std::ios::binary);
  vf.read(reinterpret_cast<char*>(values.data()), static_cast<std::streamsize>(sizeof(double) * values.size()));
  if (!vf) throw Error("values file shorter than the space");
  StrategyConfig config;
  config.id = strategy_of(argv[4]);
  config.budget = std::stoul(argv[5]);
  config.n_init = std::stoul(argv[6]);
  config.seed = std::stoull(argv[7]);
  const fs::path out = argv[8];
  std::vector<double> lambdas;
  config.inspect = [&](std::size_t, std::size_t, std::size_t, double l) { lambdas.push_back(l); };
  const Objective objective = [&](const Configuration& c) {
    const double v = values[space.position_of(c.index)];
    return std::isnan(v) ? Measurement::invalid(InvalidReason::runtime_error) : Measurement::valid(v);
  };
  const TuningRun run = run_bo(space, objective, config);
  fs::create_directories(out);
  std::vector<std::int64_t> pos;
  std::vector<double> val;
  for (const EvaluationRecord& r : run.records) {
    pos.push_back(static_cast<std::int64_t>(space.position_of(r.config_index)));
    val.push_back(r.value ? *r.value : std::numeric_limits<double>::quiet_NaN());
  }
  write_npy(out / "traj_pos.npy", pos, {pos.size()});
  write_npy(out / "traj_val.npy", val, {val.size()});
  write_npy(out / "traj_lambda.npy", lambdas, {lambdas.size()});
  std::printf("{\"n\": %zu, \"evaluations\": %zu, \"best\": %.17g, \"surrogate\": %zu, \"warnings\": %zu}\n",
              space.size(), run.evaluations, run.best_value, run.surrogate_size, run.warnings.size());
  return 0;
}

int cmd_cachegen(int argc, char** argv) {
  if (argc < 7) return 2;
  const MeasurementCache cache = make_cache(argv[2], argv[3], std::stoull(argv[4]), argv[5]);
  cache.save(argv[6]);
  std::printf("{\"entries\": %zu, \"checksum\": \"%016llx\"}\n", cache.entries.size(),
              static_cast<unsigned long long>(cache.checksum()));
  return 0;
}

// experiment <plan.json> <jobs>: the reference's own run_experiment
// (experiment.hpp:313-358) over a plan of cache files -- its thread pool of
// `jobs` workers (0 = hardware_concurrency), every run through run_strategy.
// Prints the wall time of the call (cache loading + every run) and the
// number of runs / evaluations.
int cmd_experiment(int argc, char** argv) {
  if (argc < 4) return 2;
  const fs::path plan_path = argv[2];
  const ExperimentPlan plan = ExperimentPlan::load(plan_path);
  const std::size_t jobs = std::stoul(argv[3]);
  const auto t0 = std::chrono::steady_clock::now();
  const ExperimentResult res = run_experiment(plan, jobs, plan_path.parent_path());
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::size_t runs = 0, evals = 0, failed = 0;
  for (const RunOutcome& o : res.outcomes) {
    if (o.run) {
      ++runs;
      evals += o.run->evaluations;
    } else {
      ++failed;
    }
  }
  std::printf("{\"runs\": %zu, \"failed\": %zu, \"evaluations\": %zu, \"seconds\": %.6f, \"jobs\": %zu}\n", runs,
              failed, evals, secs, jobs ? jobs : (std::size_t)std::thread::hardware_concurrency());
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_tool space|gemm|gp|runbo|bench ...\n");
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    int rc = 2;
    if (cmd == "space") rc = cmd_space(argc, argv);
    else if (cmd == "gemm") rc = cmd_gemm(argc, argv);
    else if (cmd == "gp") rc = cmd_gp(argc, argv);
    else if (cmd == "runbo") rc = cmd_runbo(argc, argv);
    else if (cmd == "runbo_spec") rc = cmd_runbo_spec(argc, argv);
    else if (cmd == "bench") rc = cmd_bench(argc, argv);
    else if (cmd == "enumjson") rc = cmd_enumjson(argc, argv);
    else if (cmd == "restrict") rc = cmd_restrict(argc, argv);
    else if (cmd == "cachegen") rc = cmd_cachegen(argc, argv);
    else if (cmd == "experiment") rc = cmd_experiment(argc, argv);
    if (rc == 2) std::fprintf(stderr, "bad arguments for %s\n", cmd.c_str());
    return rc;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
