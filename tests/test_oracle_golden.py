"""Pins the CPU oracle (oracle/gtoracle.c) before it is trusted as the checker:
against golden vectors produced by the UNMODIFIED reference
(tests/golden/*.npz, written by tests/golden/make_golden.py through
oracle/_ref/ref_tool) and against the reference's own known-answer tests
(/root/reference/proj/tests/test_gp.cpp, test_acquisition.cpp,
test_portfolio.cpp).  CPU only.
"""
import math

import numpy as np
import pytest

# ---------------------------------------------------------------- GP


def test_matern_closed_forms(oracle):
    # test_gp.cpp:24-38
    assert oracle.matern(1, 2.0, 1.0, 0.0) == 1.0
    expected = (1.0 + math.sqrt(3.0)) * math.exp(-math.sqrt(3.0))
    assert abs(oracle.matern(1, 2.0, 1.0, 2.0) - expected) <= 1e-15
    assert abs(oracle.matern(1, 2.0, 1.0, 2.0) - 0.48335) <= 1e-5
    assert oracle.matern(2, 1.0, 1.0, 50.0) < 1e-10
    assert oracle.matern(0, 0.7, 2.5, 0.0) == 2.5
    assert abs(oracle.matern(0, 0.7, 2.5, 1.4) - 2.5 * math.exp(-2.0)) <= 1e-12


def test_gp_matches_reference_golden(oracle, golden):
    g = np.load(golden / "gp_predict.npz")
    trials = sorted({k.split("_")[0] for k in g.files})
    assert len(trials) == 24
    for t in trials:
        nu, l, s2, y_mean, y_std, jitter = g[f"{t}_meta"]
        X, y, Q = g[f"{t}_X"], g[f"{t}_y"], g[f"{t}_Q"]
        rc, model = oracle.fit(int(nu), l, s2, X, y)
        assert rc == 0
        assert model["y_mean"] == pytest.approx(y_mean, rel=1e-15, abs=1e-15)
        assert model["y_std"] == pytest.approx(y_std, rel=1e-15)
        assert model["jitter"] == jitter
        mean, var = oracle.predict(model, Q)
        ref_m, ref_v = g[f"{t}_mean"], g[f"{t}_var"]
        # both follow the reference's operation order; only libm rounding differs
        np.testing.assert_allclose(mean, ref_m, rtol=0, atol=1e-9 * max(1.0, np.abs(ref_m).max()))
        np.testing.assert_allclose(var, ref_v, rtol=0, atol=1e-9 * max(1.0, s2))


def test_gp_prior_and_conditioning(oracle):
    rc, model = oracle.fit(1, 2.0, 1.7, np.zeros((0, 2)), np.zeros(0))
    assert rc == 0
    mean, var = oracle.predict(model, np.array([[0.1, 0.2], [0.5, 0.5], [0.9, 0.1]]))
    assert np.all(mean == 0.0) and np.all(var == 1.7)  # test_gp.cpp:58-70
    # identical rows, noise 0, jitter 1e-300 -> conditioning error (test_gp.cpp:235-241)
    rc, _ = oracle.fit(1, 2.0, 1.0, np.full((3, 1), 0.5), np.array([1.0, 2.0, 3.0]), noise=0.0, jitter=1e-300)
    assert rc == -2
    rc, _ = oracle.fit(1, 2.0, 1.0, np.array([[0.0], [1.0]]), np.array([1.0, np.nan]))
    assert rc == -1


# ---------------------------------------------------------------- acquisition


def test_acquisition_closed_forms(oracle):
    # test_acquisition.cpp:15-32
    assert oracle.pi(1.3, 1.0, 1.2, 0.1) == 0.5
    assert oracle.pi(2.0, 0.0, 1.0, 0.5) == 0.0
    assert oracle.pi(0.5, 0.0, 1.0, 0.5) == 1.0
    assert abs(oracle.pi(1.0 + 0.2 - 1.96 * 0.7, 0.7, 1.0, 0.2) - 0.9750021048517795) <= 1e-9
    assert oracle.ei(1.0, 0.0, 1.0, 0.0) == 0.0
    assert oracle.ei(2.0, 0.0, 1.5, 0.3) == 0.0
    assert oracle.ei(1.0, 0.0, 2.0, 0.5) == 0.5
    assert abs(oracle.ei(1.0, 1.0, 1.0, 0.0) - 0.3989422804014327) <= 1e-12
    # test_acquisition.cpp:59-63
    assert oracle.lcb(1.0, 0.5, 2.0) == 0.0
    assert oracle.lcb(1.7, 3.0, 0.0) == 1.7
    assert oracle.lcb(1.7, 0.0, 5.0) == 1.7


def test_contextual_variance(oracle):
    # test_acquisition.cpp:81-104 (state = (initial_sample_mean, initial_mean_variance))
    assert abs(oracle.cv_lambda(10.0, 1.0, 0.5, 5.0) - 0.25) <= 1e-12
    assert abs(oracle.cv_lambda(7.0, 0.42, 0.42, 7.0) - 1.0) <= 1e-12
    assert abs(oracle.cv_lambda(7.0, 0.42, 0.0, 7.0)) <= 1e-15
    assert oracle.cv_lambda(7.0, 0.42, 0.5, -1.0) is None
    assert oracle.cv_lambda(7.0, 0.42, 0.5, 0.0) is None
    assert oracle.cv_lambda(-2.0, 0.42, 0.5, 5.0) is None
    assert oracle.cv_lambda(10.0, 0.0, 0.5, 5.0) is None


def test_best_candidate_kats(oracle):
    # test_portfolio.cpp:21-40
    for af in range(3):
        assert oracle.best_candidate(af, [0.5] * 3, [1.0] * 3, 0.0, 0.0)[0] == 0
    assert oracle.best_candidate(0, [-5.0, 0.0, 1.0], [1.0] * 3, 0.0, 0.0, excluded=[1, 0, 0])[0] == 1
    assert oracle.best_candidate(0, [-5.0, 0.0, 1.0], [1.0] * 3, 0.0, 0.0, excluded=[1, 1, 1])[0] == -1
    # test_portfolio.cpp:61-71 crafted disagreement: PI -> A, EI -> B, LCB -> C
    m, s = [0.0, -2.5, -0.5], [0.1, 0.5, 1.2]
    assert oracle.best_candidate(1, m, s, 0.0, 3.0)[0] == 0
    assert oracle.best_candidate(0, m, s, 0.0, 3.0)[0] == 1
    assert oracle.best_candidate(2, m, s, 0.0, 3.0)[0] == 2
    # first-candidate rule: a NaN first score is never displaced
    assert oracle.best_candidate(2, [np.nan, -1.0], [1.0, 1.0], 0.0, 0.0)[0] == 0
    assert oracle.best_candidate(2, [1.0, np.nan, -1.0], [1.0, 1.0, 1.0], 0.0, 0.0)[0] == 2


def test_reference_trajectory_fixtures_are_consistent(golden):
    """Sanity of the committed reference trajectories: never revisit, exact
    budget accounting (test_strategies.cpp:69-82 invariants)."""
    for f in sorted(golden.glob("traj_*.npz")):
        t = np.load(f)
        pos = t["traj_pos"]
        assert len(np.unique(pos)) == len(pos), f.name
        budget = int(t["spec"][5])
        assert len(pos) == min(budget, len(t["ids"])), f.name
        vals = t["values"][pos]
        np.testing.assert_array_equal(np.isnan(vals), np.isnan(t["traj_val"]))


# ---------------------------------------------------------------- dense numpy oracle


def _np_oracle():
    import sys
    import pathlib
    sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1] / "oracle"))
    import gtoracle_np
    return gtoracle_np


def test_np_oracle_matches_reference_golden(golden):
    """oracle/gtoracle_np.py (LAPACK restatement used by the epsilon checker)
    against the reference's own GpModel::fit/predict outputs."""
    O = _np_oracle()
    g = np.load(golden / "gp_predict.npz")
    for t in sorted({k.split("_")[0] for k in g.files}):
        nu, l, s2, y_mean, y_std, jitter = g[f"{t}_meta"]
        m = O.fit(int(nu), l, s2, g[f"{t}_X"], g[f"{t}_y"])
        assert m["y_mean"] == pytest.approx(y_mean, rel=1e-14, abs=1e-14)
        assert m["y_std"] == pytest.approx(y_std, rel=1e-14)
        assert m["jitter"] == jitter
        mean, var = O.predict(m, g[f"{t}_Q"], chunk=7)
        ref_m, ref_v = g[f"{t}_mean"], g[f"{t}_var"]
        np.testing.assert_allclose(mean, ref_m, rtol=0, atol=1e-9 * max(1.0, np.abs(ref_m).max()))
        np.testing.assert_allclose(var, ref_v, rtol=0, atol=1e-9 * max(1.0, s2))


def test_np_oracle_known_answers():
    O = _np_oracle()
    # test_acquisition.cpp:15-32, 59-63, 81-104
    assert abs(float(O.acquisition(1, 1 + 0.2 - 1.96 * 0.7, 0.7, 1.0, 0.2)) - 0.9750021048517795) <= 1e-9
    assert abs(float(O.acquisition(0, 1.0, 1.0, 1.0, 0.0)) - 0.3989422804014327) <= 1e-12
    assert float(O.acquisition(0, 1.0, 0.0, 2.0, 0.5)) == 0.5 and float(O.acquisition(1, 1.0, 0.0, 0.5, 0.1)) == 0.0
    assert float(O.acquisition(2, 1.5, 0.5, 0.0, 2.0)) == -(1.5 - 2.0 * 0.5)
    assert abs(O.cv_lambda(10.0, 1.0, 0.5, 5.0) - 0.25) <= 1e-12
    assert O.cv_lambda(10.0, 1.0, 0.5, 0.0) is None and O.cv_lambda(0.0, 1.0, 0.5, 1.0) is None
    # portfolio.hpp:32-61 rule: first candidate unconditionally, ties -> lowest position, NaN never wins
    assert O.best_candidate([1.0, 3.0, 3.0, np.nan]) == 1
    assert O.best_candidate([np.nan, 3.0]) == 0
    assert O.eps_optimal([1.0, 1.0 - 5e-10, 0.5], 1) and not O.eps_optimal([1.0, 1.0 - 5e-9, 0.5], 1)
    with pytest.raises(O.ConditioningError):
        O.fit(1, 2.0, 1.0, np.full((3, 1), 0.5), np.array([1.0, 2.0, 3.0]), noise=0.0, jitter=1e-300)
