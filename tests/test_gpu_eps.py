"""Teacher-forced epsilon-optimal parity of every golden reference trajectory
(SURVEY.md §8(c) parity protocol; tests/eps_check.py): the device state is
the reference's state before every BO iteration, and the device's argmax of
every acquisition function must be epsilon-optimal (1e-9) under the dense
oracle's scores (oracle/gtoracle_np.py), with lambda within 1e-9.  This gate
does not depend on one operation order; exact trajectory identity is
asserted separately (test_gpu_trajectory.py, test_gpu_cases.py)."""
import json
import pathlib

import numpy as np
import pytest

import eps_check

pytestmark = pytest.mark.gpu

GOLD = pathlib.Path(__file__).parent / "golden"
TRAJ = sorted(GOLD.glob("traj_*.npz"))
CASES = sorted(GOLD.glob("case_*.npz"))


def _assert(rep, name):
    assert not rep.failures, f"{name}: {rep.failures[:5]}"
    assert rep.lambda_rel_err <= 1e-9, rep.lambda_rel_err
    assert rep.steps > 0


@pytest.mark.parametrize("path", TRAJ, ids=[p.stem for p in TRAJ])
def test_traj_eps_optimal(gt, path):
    t = np.load(path)
    fn, grid, sseed, inv, strat, budget, n_init, bseed = [str(x) for x in t["spec"]]
    space = gt.Space(t["coords"])
    rep = eps_check.replay(gt, space, t["coords"], t["values"], t["traj_pos"], t["traj_lambda"], strat)
    _assert(rep, path.stem)


@pytest.mark.parametrize("path", CASES, ids=[p.stem for p in CASES])
def test_case_eps_optimal(gt, path):
    t = np.load(path)
    spec = json.loads(str(t["spec"]))
    es = gt.SearchSpace([gt.ParameterDef(p["name"], p["values"]) for p in spec["params"]],
                        spec["restrictions"]).enumerate()
    np.testing.assert_array_equal(es.ids, t["ids"])
    coords = es.coords
    rep = eps_check.replay(gt, es, coords, t["values"], t["traj_pos"], t["traj_lambda"], str(t["strategy"]))
    _assert(rep, path.stem)


BIG = sorted(GOLD.glob("trajbig_*.npz"))


@pytest.mark.parametrize("path", BIG, ids=[p.stem for p in BIG])
def test_big_eps_optimal(gt, path):
    """C3 (100k candidates): every BO iteration of the reference run checked."""
    from test_gpu_trajectory import big_space
    t = np.load(path)
    coords, ids, values = big_space(t)
    rep = eps_check.replay(gt, gt.Space(coords), coords, values, t["traj_pos"], t["traj_lambda"], str(t["spec"][4]))
    _assert(rep, path.stem)
