"""Batched independent runs (gtc_run_bo_batch, run_experiment's worker model
experiment.hpp:313-358): runs driven concurrently from a host thread pool on
one device produce exactly the trajectories of the same runs one at a time
(runs share no mutable state; experiment.hpp:335-358)."""
import numpy as np
import pytest

from paper_2111_14991_b200 import synthetic

pytestmark = pytest.mark.gpu


def test_batch_equals_sequential(gt):
    coords, ids, values = synthetic.random_rough([12, 10, 8], 11, 0.3)
    space = gt.Space(coords)
    cfgs = [gt.StrategyConfig(id=sid, seed=seed, budget=60, n_init=10)
            for sid in (gt.StrategyId.bo_ei, gt.StrategyId.bo_multi, gt.StrategyId.bo_advanced_multi,
                        gt.StrategyId.bo_lcb)
            for seed in (1, 2, 3)]
    batch = gt.run_bo_batch(space, ids, cfgs, values, threads=6)
    for cfg, b in zip(cfgs, batch):
        s = gt.run_bo(space, ids, cfg, values=values)
        np.testing.assert_array_equal(b.positions, s.positions)
        np.testing.assert_array_equal(b.lambdas, s.lambdas)
        assert b.best_value == s.best_value and b.evaluations == s.evaluations


def test_batch_on_enumerated_space(gt):
    P = gt.ParameterDef
    es = gt.SearchSpace([P("bx", [1, 2, 4, 8, 16, 32, 48, 64]), P("by", [1, 2, 4, 8, 16]), P("tx", [1, 2, 3, 4, 5]),
                         P("pad", [0, 1])], ["bx * by >= 16", "tx * by < 30"]).enumerate()
    rng = np.random.default_rng(3)
    values = 1.0 + rng.random(es.n)
    values[rng.random(es.n) < 0.2] = np.nan
    cfgs = [gt.StrategyConfig(id=gt.StrategyId.bo_multi, seed=s, budget=40, n_init=8) for s in range(8)]
    batch = gt.run_bo_batch(es, es.ids, cfgs, values, threads=8)
    for cfg, b in zip(cfgs, batch):
        s = gt.run_bo(es, es.ids, cfg, values=values)
        np.testing.assert_array_equal(b.positions, s.positions)


def test_appends_across_the_shared_memory_opt_in(gt):
    """Incremental appends from 20 to 160 observations cross the point where the
    staged factor needs more than the default 48 KB of shared memory (static +
    dynamic); the appended model predicts like a full refit of the same points."""
    coords, ids, values = synthetic.random_rough([10, 10, 10, 8], 4, 0.0)
    space = gt.Space(coords)
    kern = gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0)
    rng = np.random.default_rng(9)
    pos = rng.choice(len(values), 160, replace=False)
    y = rng.random(160)
    inc = gt.SurrogateRun(space, kern, n_max=160)
    inc.fit(pos[:20], y[:20])
    for k in range(20, 160):
        inc.append(int(pos[k]), float(y[k]))
    full = gt.SurrogateRun(space, kern, n_max=160)
    full.fit(pos, y)
    m1, v1 = inc.predictions()
    m2, v2 = full.predictions()
    np.testing.assert_allclose(m1, m2, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(v1, v2, rtol=1e-9, atol=1e-9)
