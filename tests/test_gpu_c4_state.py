"""Parity in the driver-timed state (BASELINE configs[3] / bench.py C4):
N = 1,000,000 candidates (random-rough 10^6, d = 6), n = 220, bo-ei with
contextual variance, the resident loop in hold mode (gtc_run_steps with
GTC_STEPS_HOLD_N, exactly what bench.py times).  After the timed-style steps
the device posterior, lambda and pick are compared with the dense oracle
(oracle/gtoracle_np.py, gp.hpp:81-193 / acquisition.hpp / portfolio.hpp):

  * posterior mean / variance on a strided sample of 62,500 candidates within
    1e-9 (|dmu| <= 1e-9 max(|mu|, 1), |dvar| <= 1e-9 max(var, s2));
  * lambda within 1e-9 relative (the mean variance over all ~10^6 unvisited
    candidates);
  * the device pick == the oracle's best_candidate on the DEVICE posterior
    (selection bit-exact given identical inputs), and epsilon-optimal on the
    ORACLE posterior.
"""
import pathlib
import sys

import numpy as np
import pytest

import eps_check  # noqa: F401  (puts oracle/ on sys.path)
import gtoracle_np as O

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def test_c4_hold_state_matches_oracle(gt):
    import bench
    from paper_2111_14991_b200 import AcquisitionId, ContextualVarianceState, ExplorationConfig, MaternKernel, MaternNu
    cfg = bench.CONFIGS["c4"]
    coords, ids, values = bench.make_workload(cfg)
    N, n = len(values), 220
    assert N == 1_000_000
    space = gt.Space(coords)
    run = gt.SurrogateRun(space, MaternKernel(MaternNu.three_halves, 1.5, 1.0), n_max=n)
    pos = bench.prefix_positions(values, n - 1, bench.BASE_SEED)
    y = values[pos]
    run.fit(pos, y)
    for p in pos:
        run.mark_visited(int(p))
    mu_s = float(np.mean(y[:20]))
    var_s = run.mean_variance()
    cv = ContextualVarianceState(mu_s, var_s)
    expl = ExplorationConfig()
    f_base = float(np.min(y))
    run.set_values(values)
    recs = run.steps(AcquisitionId.ei, 12, f_base, expl, cv, hold=True)
    assert len(recs) == 12
    last = int(recs[-1].position)
    f_best = min(f_base, float(values[last]))
    # the state: prefix + the last step's observation at row 219, visited = prefix + last
    train = np.append(pos, last)
    model = O.fit(1, 1.5, 1.0, coords[train], values[train])
    mean_d, var_d = run.predictions()
    sample = np.arange(0, N, 16)
    m_o, v_o = O.predict(model, coords[sample])
    assert np.all(np.abs(mean_d[sample] - m_o) <= 1e-9 * np.maximum(np.abs(m_o), 1.0))
    assert np.all(np.abs(var_d[sample] - v_o) <= 1e-9 * np.maximum(v_o, 1.0))
    # full oracle posterior over the unvisited candidates (lambda, epsilon check)
    visited = np.zeros(N, dtype=bool)
    visited[train] = True
    cand = np.nonzero(~visited)[0]
    m_all, v_all = O.predict(model, coords[cand], chunk=131072)
    lam_o = O.cv_lambda(mu_s, var_s, float(np.sum(v_all)) / len(cand), f_best)
    sel = run.select([AcquisitionId.ei], f_best, expl, cv)
    assert abs(sel.lambda_ - lam_o) <= 1e-9 * max(abs(lam_o), 1.0)
    assert sel.n_candidates == len(cand)
    pick = sel.pick(AcquisitionId.ei)
    k = int(np.searchsorted(cand, pick))
    assert cand[k] == pick
    # bit-exact selection on the device's own posterior
    best_std = (f_best - model["y_mean"]) / model["y_std"]
    dev_scores = gt.acquisition_scores(AcquisitionId.ei, mean_d[cand], np.sqrt(var_d[cand]), sel.best_std,
                                       sel.lambda_)
    assert O.best_candidate(dev_scores) == k
    # epsilon-optimal on the oracle's posterior
    ora_scores = O.acquisition(0, m_all, np.sqrt(v_all), best_std, lam_o)
    assert O.eps_optimal(ora_scores, k)
    run.close()
    space.close()
