"""C1 (GEMM, bo-ei, budget 220) diagnostics: per-run wall times of
gtc_run_bo_table, and per-phase CUDA-event times of the resident loop at the
GEMM size.  Diagnostic only."""
import os
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2111_14991_b200 as gt  # noqa: E402

es, values = bench.c1_setup()
cfg = lambda r: gt.StrategyConfig(id=gt.StrategyId.bo_ei, seed=bench.BASE_SEED + r, budget=220, n_init=20)  # noqa
for r in range(3):
    gt.run_bo(es, es.ids, cfg(1000 + r), values=values)
ts = []
for r in range(20):
    t0 = time.perf_counter()
    run = gt.run_bo(es, es.ids, cfg(r), values=values)
    ts.append(1e3 * (time.perf_counter() - t0))
print("run ms:", [round(t, 1) for t in ts], "surrogate", run.surrogate_size, "evals", run.evaluations)
# phases at n = 20 .. 220 on the same space
sr = gt.SurrogateRun(es, gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0), n_max=221)
rng = np.random.default_rng(3)
valid = np.flatnonzero(~np.isnan(values))
pos = rng.choice(valid, 20, replace=False)
sr.fit(pos, values[pos])
for p in pos:
    sr.mark_visited(int(p))
sr.set_values(values)
cv = gt.ContextualVarianceState(float(np.mean(values[pos])), sr.mean_variance())
for chunk in range(4):
    recs = sr.steps(gt.AcquisitionId.ei, 50, float(np.min(values[pos])), gt.ExplorationConfig(), cv, timing=True)
    print("chunk", chunk, "steps", len(recs), "ms/step", round(sr.last_steps_ms() / max(1, len(recs)), 4),
          "phases us", [round(1e3 * x, 1) for x in sr.last_steps_phase_ms()], "exact", sr.exact_rows())
