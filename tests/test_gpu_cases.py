"""The BASELINE.json simulation-mode cases against the UNMODIFIED reference:
C1 (GEMM, 17,956 configurations: bo-ei / bo-lcb) and C2 (convolution and
pnpoly with their invalid fractions: bo-multi / bo-poi / bo-advanced-multi).
Space enumerated on the device from the same spec, same replay values; the
chosen-configuration trajectory must be identical to the reference's
(tests/golden/case_*.npz, written by tests/golden/make_golden_cases.py), with
lambda of every iteration within 1e-9 relative -- through the resident loop
(single-AF strategies) and through the per-iteration gtc_observe loop."""
import json
import pathlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = sorted(pathlib.Path(__file__).parent.joinpath("golden").glob("case_*.npz"))


def load_case(gt, path):
    t = np.load(path)
    spec = json.loads(str(t["spec"]))
    es = gt.SearchSpace([gt.ParameterDef(p["name"], p["values"]) for p in spec["params"]],
                        spec["restrictions"]).enumerate()
    np.testing.assert_array_equal(es.ids, t["ids"])  # device enumeration == reference EnumeratedSpace
    cfg = gt.StrategyConfig(id=gt.strategy_from_string(str(t["strategy"])), seed=int(t["seed"]),
                            budget=int(t["budget"]), n_init=int(t["n_init"]))
    return t, es, cfg


@pytest.mark.parametrize("resident", ["1", "0"])
@pytest.mark.parametrize("path", CASES, ids=[p.stem for p in CASES])
def test_case_trajectory_matches_reference(gt, monkeypatch, path, resident):
    monkeypatch.setenv("GTC_RESIDENT_LOOP", resident)
    t, es, cfg = load_case(gt, path)
    run = gt.run_bo(es, es.ids, cfg, values=t["values"])
    ref = t["traj_pos"]
    assert len(run.positions) == len(ref)
    first_diff = next((i for i in range(len(ref)) if run.positions[i] != ref[i]), None)
    assert first_diff is None, f"diverged at evaluation {first_diff}"
    np.testing.assert_array_equal(np.isnan(run.values), np.isnan(t["traj_val"]))
    assert run.best_value == float(t["best"])
    assert run.surrogate_size == int(t["surrogate"])
    assert run.n_warnings == int(t["warnings"])
    np.testing.assert_allclose(run.lambdas, t["traj_lambda"], rtol=1e-9, atol=1e-12)


def test_cases_batched(gt):
    """The C2 cases as one run_experiment-style batch (observe groups)."""
    for path in CASES:
        t, es, cfg = load_case(gt, path)
        out = gt.run_bo_batch(es, es.ids, [cfg, cfg], t["values"], threads=2)
        for r in out:
            np.testing.assert_array_equal(r.positions, t["traj_pos"])


@pytest.mark.parametrize("field,value,exc,msg", [
    ("lengthscale", -1.0, "Error", "kernel lengthscale must be positive"),
    ("lengthscale", 0.0, "Error", "kernel lengthscale must be positive"),
    ("discount", 1.5, "ConfigError", "discount factor must be in"),
    ("discount", 0.0, "ConfigError", "discount factor must be in"),
])
def test_out_of_range_config_fails_like_the_reference(gt, field, value, exc, msg):
    """A user-supplied lengthscale <= 0 or discount outside (0,1) is an error
    (gp.hpp:35, portfolio.hpp:107), never silently replaced by the default."""
    from paper_2111_14991_b200 import synthetic
    coords, ids, values = synthetic.random_rough([6, 6], 3, 0.0)
    space = gt.Space(coords)
    cfg = gt.StrategyConfig(id=gt.StrategyId.bo_multi, seed=1, budget=30, n_init=5, **{field: value})
    with pytest.raises(getattr(gt, exc), match=msg):
        gt.run_bo(space, ids, cfg, values=values)
