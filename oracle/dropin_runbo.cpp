// Drop-in check driver: the reference's run_bo signature executed by the B200
// library (include/gridtune_dropin/gridtune/run_bo_b200.hpp, the INTEGRATION.md
// §3 binding) on the reference's own synthetic caches (synthetic.hpp), printing
// the trajectory as JSON; tests/test_gpu_dropin.py compares it with the golden
// trajectories written by the unmodified reference (tests/golden/traj_*.npz).
//
//   dropin_runbo <function> <grid AxBx..> <space seed> <invalid|-> <strategy> <budget> <n_init> <bo seed> [ref]
// With "ref" the reference's run_bo itself runs (its GpModel / best_candidate /
// Portfolio are then the drop-in device ones too).
#include <cstdio>
#include <sstream>
#include <string>
#include <vector>

#include "gridtune/run_bo_b200.hpp"
#include "gridtune/synthetic.hpp"

using namespace gridtune;

int main(int argc, char** argv) {
  if (argc < 9) {
    std::fprintf(stderr, "usage: dropin_runbo fn grid seed invalid strategy budget n_init bo_seed [ref]\n");
    return 2;
  }
  try {
    SyntheticSpec spec;
    spec.function = argv[1];
    std::vector<std::size_t> grid;
    std::stringstream gs(argv[2]);
    for (std::string t; std::getline(gs, t, 'x');) grid.push_back(std::stoul(t));
    spec.grid = grid;
    spec.seed = std::stoull(argv[3]);
    if (std::string(argv[4]) != "-") spec.invalid_fraction = std::stod(argv[4]);
    const MeasurementCache cache = generate_synthetic(spec);
    const EnumeratedSpace space(cache.space());
    StrategyConfig config;
    config.id = *strategy_from_string(argv[5]);
    config.budget = std::stoul(argv[6]);
    config.n_init = std::stoul(argv[7]);
    config.seed = std::stoull(argv[8]);
    std::vector<double> lambdas;
    config.inspect = [&](std::size_t, std::size_t, std::size_t, double l) { lambdas.push_back(l); };
    const bool ref = argc > 9 && std::string(argv[9]) == "ref";
    const TuningRun run = ref ? run_bo(space, cache.objective(), config) : run_bo_b200(space, cache.objective(), config);
    std::printf("{\"pos\": [");
    for (std::size_t i = 0; i < run.records.size(); ++i)
      std::printf("%s%zu", i ? ", " : "", space.position_of(run.records[i].config_index));
    std::printf("], \"lambda\": [");
    for (std::size_t i = 0; i < lambdas.size(); ++i) std::printf("%s%.17g", i ? ", " : "", lambdas[i]);
    std::printf("], \"evaluations\": %zu, \"best\": %.17g, \"surrogate\": %zu, \"warnings\": %zu}\n",
                run.evaluations, run.best_value, run.surrogate_size, run.warnings.size());
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
