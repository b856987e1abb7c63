"""Exactness of the tile-pruned run selection (gtc_select / gtc_observe,
gtc_kernels.cu k_select) against the argmax of the FULL score arrays.

k_select scores exactly only candidates in tiles whose bound (from the pass's
per-tile summaries) reaches a threshold.  Here the run's resident posterior is
read back (gtc_read_predictions), every eligible candidate is scored on the
device with the same FP64 formulas (gtc_acquisition_scores) and the reference
rule is applied (portfolio.hpp:32-61: higher score, then lower position, NaN
skipped, first candidate taken unconditionally): the run selection must pick
the same position with the same score bit for bit, in early (PI saturated),
middle and late (deep-tail EI) model states, for every AF set, with and
without exclusions, and after marks that the tile summaries predate.
"""
import numpy as np
import pytest

from paper_2111_14991_b200 import synthetic

pytestmark = pytest.mark.gpu

AFS = {"ei": [0], "poi": [1], "lcb": [2], "multi": [0, 1, 2], "ei+lcb": [0, 2]}


def full_pick(gt, af, mu, var, best, lam, eligible):
    idx = np.nonzero(eligible)[0]
    s = gt.acquisition_scores(gt.AcquisitionId(af), mu[idx], np.sqrt(var[idx]), best, lam)
    if np.isnan(s[0]):
        return int(idx[0]), s[0]
    ok = ~np.isnan(s)
    top = s[ok].max()
    k = np.nonzero(ok & (s == top))[0][0]
    return int(idx[k]), top


def check_selection(gt, run, visited, f_best, cv, expl, excluded=None):
    mu, var = run.predictions()
    elig = ~visited.copy()
    if excluded is not None:
        elig[np.asarray(excluded)] = False
    for name, afs in AFS.items():
        sel = run.select([gt.AcquisitionId(a) for a in afs], f_best, expl, cv, excluded=excluded)
        assert sel.n_candidates == int(elig.sum())
        for a in afs:
            want, want_score = full_pick(gt, a, mu, var, sel.best_std, sel.lambda_, elig)
            assert sel.position[a] == want, (name, a, sel.position[a], want)
            assert sel.score[a] == want_score, (name, a)


@pytest.mark.parametrize("n_obs", [3, 40, 160])
def test_run_selection_matches_full_argmax(gt, n_obs):
    coords, ids, values = synthetic.random_rough([10, 10, 10, 10, 10], 20261017, 0.0)
    N = len(values)
    space = gt.Space(coords)
    run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.five_halves, 1.5, 1.0), n_max=200)
    rng = np.random.default_rng(n_obs)
    pos = rng.choice(N, n_obs, replace=False)
    y = values[pos]
    run.fit(pos, y)
    visited = np.zeros(N, bool)
    for p in pos:
        run.mark_visited(int(p))
        visited[p] = True
    cv = gt.ContextualVarianceState(float(np.mean(y[: min(20, n_obs)])), run.mean_variance())
    check_selection(gt, run, visited, float(np.min(y)), cv, gt.ExplorationConfig())
    check_selection(gt, run, visited, float(np.min(y)), cv,
                    gt.ExplorationConfig(gt.ExplorationConfig.Mode.constant, 0.01))
    # exclusions (duplicates and visited entries included on purpose)
    ex = list(rng.choice(N, 300, replace=False)) + list(pos[:3]) + [int(pos[0])]
    check_selection(gt, run, visited, float(np.min(y)), cv, gt.ExplorationConfig(), excluded=ex)


def test_run_selection_after_appends_and_marks(gt):
    """Incremental appends (pass-produced tile summaries), then marks without
    a pass (an invalid evaluation marks the seed candidates visited)."""
    coords, ids, values = synthetic.random_rough([12, 12, 12, 12], 5, 0.0)
    N = len(values)
    space = gt.Space(coords)
    run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0), n_max=64)
    rng = np.random.default_rng(2)
    pos = rng.choice(N, 10, replace=False)
    run.fit(pos, values[pos])
    visited = np.zeros(N, bool)
    for p in pos:
        run.mark_visited(int(p))
        visited[p] = True
    y = list(values[pos])
    cv = gt.ContextualVarianceState(float(np.mean(y)), run.mean_variance())
    expl = gt.ExplorationConfig()
    for it in range(12):
        sel = run.select([gt.AcquisitionId.ei], float(np.min(y)), expl, cv)
        p = sel.pick(gt.AcquisitionId.ei)
        if it % 3 == 2:  # invalid evaluation: mark only
            run.observe(p, None)
        else:
            run.observe(p, float(values[p]))
            y.append(float(values[p]))
        visited[p] = True
        check_selection(gt, run, visited, float(np.min(y)), cv, expl)
    # mark the current best candidates of every AF without a new pass
    for a in range(3):
        sel = run.select([gt.AcquisitionId(a)], float(np.min(y)), expl, cv)
        run.mark_visited(sel.position[a])
        visited[sel.position[a]] = True
    check_selection(gt, run, visited, float(np.min(y)), cv, expl)
