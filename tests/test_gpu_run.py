"""The resident run path (gtc_run_*): incremental bordered-Cholesky + V-row
append must equal a from-scratch refit + full predict (the reference's
fit_current + refresh_predictions, strategies.hpp:298-388) after every
append; selection must equal the reference's lambda + best_candidate
(strategies.hpp:404-436) on the same predictions."""
import numpy as np
import pytest

from paper_2111_14991_b200 import synthetic

pytestmark = pytest.mark.gpu


def rel(a, b, scale=1.0):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.maximum(np.abs(np.asarray(b)), scale)))


def make_run(gt, N=6000, d=4, nu=1, l=1.5, n_max=64, seed=0, jitter=1e-6, noise=1e-10):
    rng = np.random.default_rng(seed)
    coords = rng.random((N, d))
    space = gt.Space(coords)
    run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu(nu), l, 1.0), noise, jitter, n_max)
    return rng, coords, space, run


@pytest.mark.parametrize("nu", [0, 1, 2])
def test_incremental_append_equals_refit(gt, oracle, nu):
    rng, coords, space, run = make_run(gt, nu=nu, seed=nu)
    N = len(coords)
    order = rng.choice(N, 40, replace=False)
    y = 2.0 + rng.random(40) * 3.0
    run.fit(order[:8], y[:8])
    for k in range(8, 40):
        info = run.append(int(order[k]), float(y[k]))
        assert info.n == k + 1 and not info.rebuilt
        mean, var = run.predictions()
        rc, om = oracle.fit(nu, 1.5, 1.0, coords[order[:k + 1]], y[:k + 1])
        assert rc == 0
        assert info.jitter == om["jitter"]
        assert info.y_mean == pytest.approx(om["y_mean"], rel=1e-14)
        assert info.y_std == pytest.approx(om["y_std"], rel=1e-13)
        if k % 8 == 7 or k == 39:
            m2, v2 = oracle.predict(om, coords)
            assert rel(mean, m2) <= 1e-9, k
            assert rel(var, v2) <= 1e-9, k


def test_fit_prior_and_truncate(gt):
    rng, coords, space, run = make_run(gt, seed=5)
    info = run.fit([], [])
    mean, var = run.predictions()
    assert info.n == 0 and np.all(mean == 0.0) and np.all(var == 1.0)
    pos = rng.choice(len(coords), 12, replace=False)
    y = rng.random(12)
    run.fit(pos[:10], y[:10])
    run.append(int(pos[10]), float(y[10]))
    m1, v1 = run.predictions()
    run.append(int(pos[11]), float(y[11]))
    run.truncate(11)
    m2, v2 = run.predictions()
    assert m1.tobytes() == m2.tobytes() and v1.tobytes() == v2.tobytes()
    run.append(int(pos[11]), float(y[11]))
    run.truncate(11)
    run.append(int(pos[11]), float(y[11]))
    m3, v3 = run.predictions()
    run2 = gt.SurrogateRun(space, run.kernel, n_max=64)
    run2.fit(pos[:10], y[:10])
    run2.append(int(pos[10]), float(y[10]))
    run2.append(int(pos[11]), float(y[11]))
    m4, v4 = run2.predictions()
    assert m3.tobytes() == m4.tobytes() and v3.tobytes() == v4.tobytes()


@pytest.mark.parametrize("mode", ["constant", "contextual_variance"])
def test_select_matches_reference_step(gt, oracle, mode):
    rng, coords, space, run = make_run(gt, N=20000, d=5, seed=11)
    N = len(coords)
    pos = rng.choice(N, 30, replace=False)
    y = 1.0 + rng.random(30)
    run.fit(pos[:20], y[:20])
    for p in pos[:20]:
        run.mark_visited(int(p))
    expl = gt.ExplorationConfig(gt.ExplorationConfig.Mode[mode])
    cv = gt.ContextualVarianceState(float(np.mean(y[:20])), run.mean_variance())
    visited = np.zeros(N, bool)
    visited[pos[:20]] = True
    for k in range(20, 30):
        mean, var = run.predictions()
        cand = np.nonzero(~visited)[0]
        mv = oracle.mean(var[cand])
        assert abs(run.mean_variance() - mv) <= 1e-12 * mv
        fb = float(np.min(y[:k]))
        lam = expl.constant
        if mode == "contextual_variance":
            lam = oracle.cv_lambda(cv.initial_sample_mean, cv.initial_mean_variance, mv, fb)
        sel = run.select(list(gt.AcquisitionId), fb, expl, cv)
        assert sel.n_candidates == len(cand)
        assert abs(sel.lambda_ - lam) <= 1e-12 * max(lam, 1e-300)
        best_std = (fb - np.mean(y[:k])) / np.std(y[:k])
        assert abs(sel.best_std - best_std) <= 1e-12 * max(1.0, abs(best_std))
        for af in gt.AcquisitionId:
            p, s = oracle.best_candidate(int(af), mean[cand], np.sqrt(var[cand]), sel.best_std, sel.lambda_)
            assert sel.pick(af) == cand[p], (k, af)
        run.mark_visited(int(pos[k]))
        visited[pos[k]] = True
        run.append(int(pos[k]), float(y[k]))


def test_select_exclusions_and_exhaustion(gt):
    rng, coords, space, run = make_run(gt, N=300, d=2, seed=3)
    run.fit([0, 1], [1.0, 2.0])
    sel = run.select([gt.AcquisitionId.ei], 1.0, gt.ExplorationConfig(gt.ExplorationConfig.Mode.constant))
    p = sel.pick(gt.AcquisitionId.ei)
    sel2 = run.select([gt.AcquisitionId.ei], 1.0, gt.ExplorationConfig(gt.ExplorationConfig.Mode.constant),
                      excluded=[p])
    assert sel2.pick(gt.AcquisitionId.ei) != p and sel2.n_candidates == 299
    for j in range(300):
        run.mark_visited(j)
    assert run.unvisited_count() == 0
    with pytest.raises(gt.Error, match="no candidates remaining"):
        run.select([gt.AcquisitionId.ei], 1.0)


def test_append_jitter_escalation_matches_refit(gt, oracle):
    """A near-duplicate candidate makes the bordered pivot fail at the base
    jitter; the run refactorises with doubled jitter like gp.hpp:116-129."""
    coords = np.array([[0.2, 0.2], [0.2 + 1e-9, 0.2], [0.7, 0.1], [0.9, 0.9], [0.5, 0.5]])
    space = gt.Space(coords)
    run = gt.SurrogateRun(space, gt.MaternKernel(), 0.0, 1e-17, 8)
    run.fit([0, 2], [1.0, 3.0])
    info = run.append(1, 2.0)
    assert info.rebuilt
    rc, om = oracle.fit(1, 2.0, 1.0, coords[[0, 2, 1]], np.array([1.0, 3.0, 2.0]), noise=0.0, jitter=1e-17)
    assert rc == 0 and info.jitter == om["jitter"] == 1.6e-16
    run.append(3, 0.5)  # continues incrementally at the escalated jitter
    rc, om = oracle.fit(1, 2.0, 1.0, coords[[0, 2, 1, 3]], np.array([1.0, 3.0, 2.0, 0.5]), noise=0.0, jitter=1e-17)
    mean, var = run.predictions()
    m2, v2 = oracle.predict(om, coords)
    assert rel(var[[3, 4]], v2[[3, 4]]) <= 1e-6


def test_truncate_after_escalation_refits_prefix_at_base_jitter(gt, oracle):
    """Truncating below the observation that forced a jitter escalation gives
    GpModel::fit of the prefix, which restarts at the base jitter."""
    coords = np.array([[0.2, 0.2], [0.2 + 1e-9, 0.2], [0.7, 0.1], [0.9, 0.9], [0.5, 0.5]])
    run = gt.SurrogateRun(gt.Space(coords), gt.MaternKernel(), 0.0, 1e-17, 8)
    run.fit([0, 2], [1.0, 3.0])
    assert run.append(1, 2.0).jitter == 1.6e-16
    info = run.truncate(2)
    assert info.jitter == 1e-17 and info.n == 2
    rc, om = oracle.fit(1, 2.0, 1.0, coords[[0, 2]], np.array([1.0, 3.0]), noise=0.0, jitter=1e-17)
    mean, var = run.predictions()
    m2, v2 = oracle.predict(om, coords)
    assert rel(mean, m2) <= 1e-9 and rel(var, v2) <= 1e-9
    info = run.append(3, 0.5)  # appends at the base jitter again
    assert info.jitter == 1e-17


def test_conditioning_error_on_append(gt):
    coords = np.array([[0.5], [0.5 + 1e-12], [0.9]])
    run = gt.SurrogateRun(gt.Space(coords), gt.MaternKernel(), 0.0, 1e-300, 8)
    run.fit([0], [1.0])
    with pytest.raises(gt.ModelConditioningError, match="jitter escalation"):
        run.append(1, 2.0)


def test_rescaling_invariance_is_bitwise(gt):
    """Power-of-two rescaling of the observations leaves standardized
    predictions and picks bit-identical (test_strategies.cpp:274-295)."""
    coords, ids, values = synthetic.random_rough([20, 20, 10], 41, 0.0)
    space = gt.Space(coords)
    rng = np.random.default_rng(2)
    pos = rng.choice(len(coords), 25, replace=False)
    outs = []
    for scale in (1.0, 2.0, 0.25, 1024.0):
        run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.three_halves, 1.5), n_max=32)
        y = values[pos] * scale
        run.fit(pos[:20], y[:20])
        for p in pos[:20]:
            run.mark_visited(int(p))
        cv = gt.ContextualVarianceState(float(np.mean(y[:20])), run.mean_variance())
        picks = []
        for k in range(20, 25):
            sel = run.select(list(gt.AcquisitionId), float(np.min(y[:k])), gt.ExplorationConfig(), cv)
            picks.append(sel.position)
            run.mark_visited(int(pos[k]))
            run.append(int(pos[k]), float(y[k]))
        mean, var = run.predictions()
        outs.append((mean.tobytes(), var.tobytes(), picks))
    for o in outs[1:]:
        assert o == outs[0]


def test_c4_scale_append_vs_oracle_sample(gt, oracle):
    """N = 1M candidates (C4 shape), n = 60: device posterior after an append
    equals the oracle refit on a strided sample of 20k candidates."""
    coords, ids, values = synthetic.random_rough([10] * 6, 20261017, 0.0)
    space = gt.Space(coords)
    run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.three_halves, 1.5), n_max=64)
    rng = np.random.default_rng(4)
    pos = rng.choice(len(coords), 60, replace=False)
    run.fit(pos[:59], values[pos[:59]])
    run.append(int(pos[59]), float(values[pos[59]]))
    mean, var = run.predictions()
    rc, om = oracle.fit(1, 1.5, 1.0, coords[pos], values[pos])
    sample = np.arange(0, len(coords), 50)
    m2, v2 = oracle.predict(om, coords[sample])
    assert rel(mean[sample], m2) <= 1e-9
    assert rel(var[sample], v2) <= 1e-9


def test_observe_equals_separate_calls(gt):
    """gtc_observe (one round trip) == mark_visited + append + select, bitwise,
    for valid and invalid observations."""
    rng, coords, space, run_a = make_run(gt, N=30000, d=5, seed=21)
    run_b = gt.SurrogateRun(space, run_a.kernel, n_max=64)
    pos = rng.choice(len(coords), 40, replace=False)
    y = 1.0 + rng.random(40)
    for r in (run_a, run_b):
        r.fit(pos[:20], y[:20])
        for p in pos[:20]:
            r.mark_visited(int(p))
    cv = gt.ContextualVarianceState(float(np.mean(y[:20])), run_a.mean_variance())
    afs = list(gt.AcquisitionId)
    fb = float(np.min(y[:20]))
    for k in range(20, 40):
        valid = k % 3 != 0
        fb = min(fb, float(y[k])) if valid else fb
        info, sa = run_a.observe(int(pos[k]), float(y[k]) if valid else None, afs, fb, gt.ExplorationConfig(), cv)
        run_b.mark_visited(int(pos[k]))
        if valid:
            run_b.append(int(pos[k]), float(y[k]))
        sb = run_b.select(afs, fb, gt.ExplorationConfig(), cv)
        assert sa.position == sb.position and sa.lambda_ == sb.lambda_ and sa.score == sb.score
        assert sa.n_candidates == sb.n_candidates == run_a.unvisited_count()
        ma, va = run_a.predictions()
        mb, vb = run_b.predictions()
        assert ma.tobytes() == mb.tobytes() and va.tobytes() == vb.tobytes()


def test_async_truncate_defers_but_matches_eager(gt):
    """gtc_truncate without info defers the prefix standardisation/beta to the
    first consumer; predictions, the mean variance and a following append
    equal the eager truncate's bit for bit."""
    rng = np.random.default_rng(21)
    coords = rng.random((5000, 3))
    pos = rng.choice(5000, 30, replace=False)
    y = rng.standard_normal(30) * 2.0 + 5.0

    def make():
        run = gt.SurrogateRun(gt.Space(coords), gt.MaternKernel(gt.MaternNu.five_halves, 0.9, 1.2), n_max=40)
        run.fit(pos[:25], y[:25])
        return run

    a, b = make(), make()
    a.truncate(18)
    b.truncate_async(18)
    ma, va = a.predictions()
    mb, vb = b.predictions()
    np.testing.assert_array_equal(ma, mb)
    np.testing.assert_array_equal(va, vb)
    assert a.mean_variance() == b.mean_variance()
    # truncate, then append right away (the append recomputes the statistics)
    c, e = make(), make()
    c.truncate(20)
    e.truncate_async(20)
    c.append(int(pos[27]), float(y[27]))
    e.append(int(pos[27]), float(y[27]))
    mc, vc = c.predictions()
    me, ve = e.predictions()
    np.testing.assert_array_equal(mc, me)
    np.testing.assert_array_equal(vc, ve)
    # a refit after an async truncate starts from clean statistics
    e.truncate_async(10)
    e.fit(pos[:12], y[:12])
    c.fit(pos[:12], y[:12])
    np.testing.assert_array_equal(c.predictions()[0], e.predictions()[0])
