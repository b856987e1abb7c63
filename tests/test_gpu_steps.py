"""Resident BO loop (gtc_run_steps, simulation mode): k iterations of a
single-AF strategy on the device must equal the gtc_observe loop driven from
the host -- the run_bo iteration of strategies.hpp:401-449 -- pick for pick,
lambda for lambda and posterior bit for bit (same kernels, per-step inputs
read from the loop state instead of launch arguments)."""
import numpy as np
import pytest

from paper_2111_14991_b200 import synthetic

pytestmark = pytest.mark.gpu


def setup(gt, grid, invalid, seed, nu=1, n_init=20, n_max=160, l=1.5):
    coords, ids, values = synthetic.random_rough(grid, seed, invalid)
    space = gt.Space(coords)
    run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu(nu), l, 1.0), 1e-10, 1e-6, n_max)
    rng = np.random.default_rng(seed)
    valid = np.nonzero(~np.isnan(values))[0]
    init = rng.choice(valid, n_init, replace=False)
    run.fit(init, values[init])
    for p in init:
        run.mark_visited(int(p))
    cv = gt.ContextualVarianceState(float(np.mean(values[init])), run.mean_variance())
    return space, run, values, init, cv


def host_loop(gt, run, values, af, k, f_best, expl, cv):
    """The gtc_observe loop: select -> evaluate -> observe (+ next selection)."""
    picks, lams, fbs = [], [], []
    sel = run.select([af], f_best, expl, cv)
    for _ in range(k):
        if sel.n_candidates == 0:
            break
        p = sel.pick(af)
        y = values[p]
        picks.append(p)
        lams.append(sel.lambda_)
        valid = not np.isnan(y)
        if valid:
            f_best = min(f_best, float(y))
        _, sel = run.observe(p, float(y) if valid else None, [af], f_best, expl, cv)
        fbs.append(f_best)
    return picks, lams


@pytest.mark.parametrize("af", [0, 1, 2])
@pytest.mark.parametrize("mode", ["cv", "const"])
def test_steps_equal_observe_loop(gt, af, mode):
    af = gt.AcquisitionId(af)
    expl = gt.ExplorationConfig() if mode == "cv" else gt.ExplorationConfig(gt.ExplorationConfig.Mode.constant, 0.01)
    grid, inv, seed, k = [8, 8, 8, 6], 0.3, 11 + int(af), 90
    space, run_a, values, init, cv = setup(gt, grid, inv, seed)
    f0 = float(np.min(values[init]))
    picks_h, lams_h = host_loop(gt, run_a, values, af, k, f0, expl, cv)
    m_h, v_h = run_a.predictions()

    _, run_b, _, _, cv_b = setup(gt, grid, inv, seed)
    assert cv_b.initial_mean_variance == cv.initial_mean_variance
    run_b.set_values(values)
    recs = run_b.steps(af, k, f0, expl, cv)
    picks_d = [r.position for r in recs]
    assert picks_d == picks_h
    np.testing.assert_array_equal([r.lambda_ for r in recs], lams_h)
    vals = values[picks_d]
    np.testing.assert_array_equal([bool(r.valid) for r in recs], ~np.isnan(vals))
    assert any(not r.valid for r in recs)  # the invalid (O(1) total update) path ran
    m_d, v_d = run_b.predictions()
    np.testing.assert_array_equal(m_d, m_h)
    np.testing.assert_array_equal(v_d, v_h)
    assert run_b.unvisited_count() == run_a.unvisited_count()
    # continuing from the host API after a resident chunk: same next selection
    fb = min([f0] + [float(v) for v in vals if not np.isnan(v)])
    s_a = run_a.select([af], fb, expl, cv)
    s_b = run_b.select([af], fb, expl, cv)
    assert s_a.pick(af) == s_b.pick(af) and s_a.lambda_ == s_b.lambda_


def test_steps_chunked_and_nu(gt):
    """Several calls in a row (host state re-synchronised between chunks) and
    the other Matern orders."""
    for nu in (0, 2):
        af = gt.AcquisitionId.ei
        expl = gt.ExplorationConfig()
        space, run_a, values, init, cv = setup(gt, [10, 10, 6, 5], 0.2, 3 + nu, nu=nu)
        f0 = float(np.min(values[init]))
        picks_h, _ = host_loop(gt, run_a, values, af, 70, f0, expl, cv)
        _, run_b, _, _, _ = setup(gt, [10, 10, 6, 5], 0.2, 3 + nu, nu=nu)
        run_b.set_values(values)
        picks_d, fb = [], f0
        for k in (1, 9, 25, 35):
            recs = run_b.steps(af, k, fb, expl, cv)
            picks_d += [r.position for r in recs]
            fb = min([fb] + [r.value for r in recs if r.valid])
        assert picks_d == picks_h


def test_steps_exhaust_space(gt):
    """A space smaller than the chunk: the device loop stops when every
    candidate has been visited (run_bo's exhaustion, strategies.hpp:399)."""
    af = gt.AcquisitionId.lcb
    space, run, values, init, cv = setup(gt, [5, 4, 3], 0.25, 5, n_max=80)
    run.set_values(values)
    recs = run.steps(af, 200, float(np.min(values[init])), gt.ExplorationConfig(), cv)
    assert len(recs) == 60 - 20
    assert sorted([r.position for r in recs] + list(init)) == list(range(60))
    assert run.unvisited_count() == 0


def test_steps_hold_equals_rollback_loop(gt):
    """GTC_STEPS_HOLD_N (the bench's steady state) == the host rollback loop
    (truncate to n0, observe, unmark the pick)."""
    af = gt.AcquisitionId.ei
    expl = gt.ExplorationConfig()
    grid, seed, k = [10, 10, 10, 8], 21, 40
    space, run_a, values, init, cv = setup(gt, grid, 0.0, seed, n_init=60, n_max=64)
    f0 = float(np.min(values[init]))
    n0 = 60
    pick = run_a.select([af], f0, expl, cv).pick(af)
    picks_h = []
    for _ in range(k):
        run_a.truncate_async(n0)
        picks_h.append(pick)
        y = float(values[pick])
        _, s = run_a.observe(pick, y, [af], min(f0, y), expl, cv)
        run_a.unmark_visited(pick)
        pick = s.pick(af)
    _, run_b, _, _, _ = setup(gt, grid, 0.0, seed, n_init=60, n_max=64)
    run_b.set_values(values)
    recs = run_b.steps(af, k, f0, expl, cv, hold=True)
    assert [r.position for r in recs] == picks_h
    # both models now hold the init points + the last pick at row n0
    m_a, v_a = run_a.predictions()
    m_b, v_b = run_b.predictions()
    np.testing.assert_array_equal(m_a, m_b)
    np.testing.assert_array_equal(v_a, v_b)
    # the host path unmarked the last pick too; the device run keeps it visited
    assert run_b.unvisited_count() == run_a.unvisited_count() - 1


@pytest.mark.parametrize("variant", ["cv", "const", "free_invalid", "nu52"])
def test_run_bo_resident_equals_observe_loop(gt, monkeypatch, variant):
    """gtc_run_bo_table with the resident loop == the per-iteration gtc_observe
    loop (GTC_RESIDENT_LOOP=0), every BO strategy (the portfolio of bo-multi /
    bo-advanced-multi on the device vs the host Portfolio)."""
    coords, ids, values = synthetic.random_rough([12, 10, 8], 7, 0.3)
    space = gt.Space(coords)
    for sid in (gt.StrategyId.bo_ei, gt.StrategyId.bo_poi, gt.StrategyId.bo_lcb, gt.StrategyId.bo_multi,
                gt.StrategyId.bo_advanced_multi):
        cfg = gt.StrategyConfig(id=sid, seed=5 + int(sid), budget=120, n_init=10)
        if variant == "const":
            cfg.exploration = gt.ExplorationConfig(gt.ExplorationConfig.Mode.constant, 0.05)
        elif variant == "free_invalid":
            cfg.invalid_consumes_budget = False
        elif variant == "nu52":
            cfg.nu = gt.MaternNu.five_halves
        monkeypatch.setenv("GTC_RESIDENT_LOOP", "0")
        a = gt.run_bo(space, ids, cfg, values=values)
        monkeypatch.setenv("GTC_RESIDENT_LOOP", "1")
        b = gt.run_bo(space, ids, cfg, values=values)
        np.testing.assert_array_equal(a.positions, b.positions)
        np.testing.assert_array_equal(a.lambdas, b.lambdas)
        assert (a.evaluations, a.budget_consumed, a.invalid_count, a.surrogate_size, a.n_warnings) == \
               (b.evaluations, b.budget_consumed, b.invalid_count, b.surrogate_size, b.n_warnings)
        assert a.best_value == b.best_value


def test_batch_resident_equals_groups(gt, monkeypatch):
    """gtc_run_bo_batch: single-AF runs resident (default) or in observe groups
    (GTC_BATCH_RESIDENT=0), mixed with multi-AF runs -- identical runs."""
    coords, ids, values = synthetic.random_rough([12, 10, 8], 13, 0.3)
    space = gt.Space(coords)
    cfgs = [gt.StrategyConfig(id=sid, seed=seed, budget=80, n_init=10)
            for sid in (gt.StrategyId.bo_ei, gt.StrategyId.bo_multi, gt.StrategyId.bo_poi, gt.StrategyId.bo_lcb,
                        gt.StrategyId.bo_advanced_multi)
            for seed in (1, 2, 3, 4)]
    monkeypatch.setenv("GTC_BATCH_RESIDENT", "0")
    a = gt.run_bo_batch(space, ids, cfgs, values, threads=8)
    monkeypatch.setenv("GTC_BATCH_RESIDENT", "1")
    b = gt.run_bo_batch(space, ids, cfgs, values, threads=8)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x.positions, y.positions)
        np.testing.assert_array_equal(x.lambdas, y.lambdas)


@pytest.mark.parametrize("mode", [1, 2])
def test_portfolio_skips_and_promotions(gt, monkeypatch, mode):
    """Long portfolio runs whose duplicate counters / bands fire (small skip
    threshold): the device portfolio deactivates and promotes exactly like the
    host Portfolio (portfolio.hpp:191-299)."""
    coords, ids, values = synthetic.random_rough([10, 10, 8, 6], 17, 0.25)
    space = gt.Space(coords)
    sid = gt.StrategyId.bo_multi if mode == 1 else gt.StrategyId.bo_advanced_multi
    for seed, skip in ((1, 1), (2, 2), (3, 5)):
        cfg = gt.StrategyConfig(id=sid, seed=seed, budget=200, n_init=15, skip_threshold=skip)
        monkeypatch.setenv("GTC_RESIDENT_LOOP", "0")
        a = gt.run_bo(space, ids, cfg, values=values)
        monkeypatch.setenv("GTC_RESIDENT_LOOP", "1")
        b = gt.run_bo(space, ids, cfg, values=values)
        np.testing.assert_array_equal(a.positions, b.positions)
        np.testing.assert_array_equal(a.lambdas, b.lambdas)


def test_resident_jitter_escalation_equals_observe_loop(gt, monkeypatch):
    """Duplicated configurations (identical coordinates) make bordered pivots
    fail at a tiny jitter: the resident loop halts on the device, the host
    refactorises with escalated jitter (gp.hpp:116-129) and continues -- same
    trajectory as the per-iteration loop, every strategy."""
    rng = np.random.default_rng(4)
    base = rng.random((300, 3))
    coords = np.repeat(base, 4, axis=0)                 # every configuration 4 times
    ids = np.arange(len(coords), dtype=np.uint64)
    values = 1.0 + rng.random(len(coords))
    values[rng.random(len(coords)) < 0.1] = np.nan
    space = gt.Space(coords)
    for sid in (gt.StrategyId.bo_ei, gt.StrategyId.bo_multi, gt.StrategyId.bo_advanced_multi):
        cfg = gt.StrategyConfig(id=sid, seed=3, budget=90, n_init=10, noise=0.0, jitter=1e-13)
        monkeypatch.setenv("GTC_RESIDENT_LOOP", "0")
        a = gt.run_bo(space, ids, cfg, values=values)
        monkeypatch.setenv("GTC_RESIDENT_LOOP", "1")
        b = gt.run_bo(space, ids, cfg, values=values)
        np.testing.assert_array_equal(a.positions, b.positions)
        np.testing.assert_array_equal(a.lambdas, b.lambdas)
        assert a.surrogate_size == b.surrogate_size


def test_resident_pivot_failure_refit(gt):
    """Only duplicates of training points left as candidates: the bordered
    pivot fails on the device, the chunk halts, the host refactorises with
    escalated jitter and the loop continues -- same picks, posterior and
    outcome (or the same ModelConditioningError) as the gtc_observe loop."""
    rng = np.random.default_rng(8)
    uniq = rng.random((40, 3))
    coords = np.concatenate([uniq, uniq[:10]])          # positions 40..49 duplicate 0..9
    values = 1.0 + rng.random(len(coords))
    values[40:] = values[:10]

    def make():
        space = gt.Space(coords)
        run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0), 0.0, 1e-16, 64)
        run.fit(np.arange(10), values[:10])
        for p in range(40):                             # only the duplicates stay candidates
            run.mark_visited(p)
        return space, run

    expl = gt.ExplorationConfig(gt.ExplorationConfig.Mode.constant, 0.01)
    cv = gt.ContextualVarianceState()
    f0 = float(np.min(values[:10]))
    _, run_a = make()
    af = gt.AcquisitionId.ei
    picks_h, jitters, err_h = [], [], None
    try:
        sel = run_a.select([af], f0, expl, cv)
        for _ in range(6):
            p = sel.pick(af)
            picks_h.append(p)
            info, sel = run_a.observe(p, float(values[p]), [af], f0, expl, cv)
            jitters.append(info.jitter)
    except gt.ModelConditioningError as e:
        picks_h, err_h = None, str(e)
    assert err_h is not None or max(jitters) > 1e-16  # the escalation path ran
    _, run_b = make()
    run_b.set_values(values)
    try:
        recs = run_b.steps(gt.AcquisitionId.ei, 6, f0, expl, cv)
        err_d = None
    except gt.ModelConditioningError as e:
        recs, err_d = None, str(e)
    assert err_d == err_h
    if err_h is None:
        assert [r.position for r in recs] == picks_h
        m_a, v_a = run_a.predictions()
        m_b, v_b = run_b.predictions()
        np.testing.assert_array_equal(m_a, m_b)
        np.testing.assert_array_equal(v_a, v_b)


@pytest.mark.parametrize("portfolio", [0, 1, 2])
def test_graph_launched_chunks(gt, portfolio):
    """Without PDL gtc_run_steps launches captured graphs (16 iterations, then
    single iterations); same picks and posterior as PDL launches, across
    chunk sizes that reuse and re-capture the graphs."""
    af = gt.AcquisitionId.ei
    expl = gt.ExplorationConfig()
    out = []
    for pdl in (True, False):
        space, run, values, init, cv = setup(gt, [10, 10, 6, 5], 0.2, 31)
        run.set_values(values)
        run.set_pdl(pdl)
        if portfolio:
            run.set_portfolio(portfolio, 2, 0.65 if portfolio == 1 else 0.75, 0.1)
        picks, fb = [], float(np.min(values[init]))
        for k in (20, 17, 1, 45, 16):
            recs = run.steps(af, k, fb, expl, cv)
            picks += [(r.position, r.by, r.lambda_) for r in recs]
            fb = min([fb] + [r.value for r in recs if r.valid])
        out.append((picks, run.predictions()))
    assert out[0][0] == out[1][0]
    np.testing.assert_array_equal(out[0][1][0], out[1][1][0])
    np.testing.assert_array_equal(out[0][1][1], out[1][1][1])


def test_steps_argument_errors(gt):
    """gtc_run_steps preconditions map to the reference error types."""
    af = gt.AcquisitionId.ei
    expl = gt.ExplorationConfig()
    space, run, values, init, cv = setup(gt, [6, 6, 5], 0.0, 2, n_max=40)
    f0 = float(np.min(values[init]))
    with pytest.raises(gt.Error, match="no value table"):
        run.steps(af, 3, f0, expl, cv)
    run.set_values(values)
    a, _ = run._args([gt.AcquisitionId.ei, gt.AcquisitionId.lcb], f0, expl, cv, None)
    import ctypes as C
    from paper_2111_14991_b200 import _lib
    recs = (_lib.gtc_step_record * 4)()
    done = C.c_int32()
    info = _lib.gtc_fit_info()
    rc = gt.load().gtc_run_steps(run.handle, C.byref(a), 4, 0, recs, C.byref(done), C.byref(info))
    assert rc == _lib.GTC_ERR_INVALID and b"exactly one" in gt.load().gtc_last_error()
    run.set_portfolio(1)
    with pytest.raises(gt.Error, match="single-AF"):
        run.steps(af, 3, f0, expl, cv, hold=True)
    with pytest.raises(gt.ConfigError):
        run.set_portfolio(1, skip_threshold=0)
    with pytest.raises(gt.ConfigError):
        run.set_portfolio(2, discount=1.0)
    # capacity: the model cannot grow past n_max (20 initial + 20 appended)
    run.set_portfolio(0)
    with pytest.raises(gt.Error, match="n_max"):
        run.steps(af, 30, f0, expl, cv)


def test_steps_hold_with_invalid_values(gt):
    """GTC_STEPS_HOLD_N with runtime-invalid values (the C3 bench): an invalid
    pick is marked and stays visited without touching the model; a valid one
    replaces the observation at row n0 and un-marks the position it replaces.
    Same picks as that protocol driven through gtc_observe from the host."""
    af = gt.AcquisitionId.lcb
    expl = gt.ExplorationConfig()
    grid, seed, k = [10, 10, 10, 8], 23, 60
    space, run_a, values, init, cv = setup(gt, grid, 0.3, seed, n_init=60, n_max=64)
    f0 = float(np.min(values[init]))
    n0 = 60
    sel = run_a.select([af], f0, expl, cv)
    picks_h, prev = [], None
    for _ in range(k):
        p = sel.pick(af)
        picks_h.append(p)
        y = values[p]
        if np.isnan(y):
            _, sel = run_a.observe(p, None, [af], f0 if prev is None else min(f0, values[prev]), expl, cv)
            continue
        run_a.truncate_async(n0)
        if prev is not None:
            run_a.unmark_visited(prev)
        prev = p
        _, sel = run_a.observe(p, float(y), [af], min(f0, float(y)), expl, cv)
    _, run_b, _, _, _ = setup(gt, grid, 0.3, seed, n_init=60, n_max=64)
    run_b.set_values(values)
    recs = run_b.steps(af, k, f0, expl, cv, hold=True)
    assert any(not r.valid for r in recs)
    assert [r.position for r in recs] == picks_h
