"""Teacher-forced epsilon-optimal trajectory checker (SURVEY.md §8(c) parity
protocol) — TEST INFRASTRUCTURE.

Replays a reference run_bo trajectory (strategies.hpp:261-457) step by step
through the device's per-iteration API (gtc_fit / gtc_select / gtc_observe):
before every BO iteration the device state is the reference's state (same
training set, same visited set -- the reference's picks are fed back, not
the device's), and

  * the device's lambda (strategies.hpp:404-418) matches the oracle's within
    1e-9 relative;
  * every acquisition function's device argmax is epsilon-optimal under the
    oracle's scores: score(pick) >= best - 1e-9 * max(|best|, 1) -- so it is
    the oracle's argmax exactly wherever the oracle's top-2 gap exceeds that
    band;
  * the reference's own pick is epsilon-optimal under the oracle's scores for
    (one of) the function(s) that could have produced it -- the check of the
    oracle against the reference.

The oracle is oracle/gtoracle_np.py (dense LAPACK restatement of gp.hpp /
acquisition.hpp / portfolio.hpp), so exact identity to one particular
operation order (the shim-built reference's) is not what is gated here.
"""
from __future__ import annotations

import pathlib
import sys
from dataclasses import dataclass, field

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
import gtoracle_np as O  # noqa: E402

EPS = 1e-9
AFS = {"bo-ei": (0,), "bo-poi": (1,), "bo-lcb": (2,), "bo-multi": (0, 1, 2), "bo-advanced-multi": (0, 1, 2)}


@dataclass
class Report:
    steps: int = 0
    exact: int = 0              # device argmax == oracle argmax (every AF)
    eps_only: int = 0           # differed from the oracle's argmax, but within the band
    lambda_rel_err: float = 0.0
    failures: list = field(default_factory=list)


def replay(gt, space, coords, values, traj_pos, traj_lambda, strategy: str, nu: int = 1,
           lengthscale: float = 1.5, s2: float = 1.0, noise: float = 1e-10, jitter: float = 1e-6,
           steps=None) -> Report:
    """`space`: the device Space (or EnumeratedSpace) over `coords`.  `steps`:
    optional subset of BO-iteration indices to check (all by default; the
    device state is advanced through every step either way)."""
    from paper_2111_14991_b200 import (AcquisitionId, ContextualVarianceState, ExplorationConfig, MaternKernel,
                                       MaternNu)
    afs = AFS[strategy]
    N = len(values)
    n0 = len(traj_pos) - len(traj_lambda)          # initial-design evaluations (sampling.hpp:73-160)
    init = [int(p) for p in traj_pos[:n0]]
    train = [p for p in init if not np.isnan(values[p])]
    run = gt.SurrogateRun(space, MaternKernel(MaternNu(nu), lengthscale, s2), noise=noise, jitter=jitter,
                          n_max=max(len(train) + len(traj_lambda), 2))
    visited = np.zeros(N, dtype=bool)
    for p in init:
        run.mark_visited(p)
        visited[p] = True
    run.fit(train, values[train])
    model = O.fit(nu, lengthscale, s2, coords[train], values[train], noise, jitter)
    mu_s = sum(float(values[p]) for p in train) / len(train)      # InitialSample::mean_observation
    cand = np.nonzero(~visited)[0]
    _, var0 = O.predict(model, coords[cand])
    var_s_oracle = float(np.sum(var0)) / len(cand)                # strategies.hpp:392-397
    var_s = run.mean_variance()
    rep = Report()
    rep.lambda_rel_err = abs(var_s - var_s_oracle) / max(abs(var_s_oracle), 1e-300)
    cv = ContextualVarianceState(mu_s, var_s)
    expl = ExplorationConfig()
    f_best = min(float(values[p]) for p in train)
    check = set(range(len(traj_lambda))) if steps is None else set(steps)
    for t in range(len(traj_lambda)):
        pick = int(traj_pos[n0 + t])
        if t in check:
            assert model is not None
            sel = run.select([AcquisitionId(a) for a in afs], f_best, expl, cv)
            cand = np.nonzero(~visited)[0]
            mean, var = O.predict(model, coords[cand])
            lam = O.cv_lambda(mu_s, var_s_oracle, float(np.sum(var)) / len(cand), f_best)
            lam = expl.constant if lam is None else lam
            rel = abs(sel.lambda_ - lam) / max(abs(lam), 1.0)
            rep.lambda_rel_err = max(rep.lambda_rel_err, rel)
            if abs(sel.lambda_ - traj_lambda[t]) > 1e-9 * max(abs(traj_lambda[t]), 1.0):
                rep.failures.append((t, "lambda vs reference", sel.lambda_, float(traj_lambda[t])))
            best_std = O.standardize(model, f_best)
            sd = np.sqrt(var)
            same = True
            ref_ok = False
            for af in afs:
                scores = O.acquisition(af, mean, sd, best_std, lam)
                dev = int(sel.position[af])
                k = int(np.searchsorted(cand, dev))
                if k >= len(cand) or cand[k] != dev:
                    rep.failures.append((t, f"af{af} picked a visited position", dev))
                    continue
                ob = O.best_candidate(scores)
                if k != ob:
                    same = False
                    if not O.eps_optimal(scores, k, EPS):
                        rep.failures.append((t, f"af{af} not eps-optimal", dev, float(scores[k]),
                                             int(cand[ob]), float(scores[ob])))
                kr = int(np.searchsorted(cand, pick))
                ref_ok |= O.eps_optimal(scores, kr, EPS)
            if not ref_ok:
                rep.failures.append((t, "reference pick not eps-optimal under the oracle", pick))
            rep.steps += 1
            rep.exact += same
            rep.eps_only += not same
        # feed the reference's evaluation back (teacher forcing)
        y = values[pick]
        visited[pick] = True
        if np.isnan(y):
            run.observe(pick, None)
        else:
            run.observe(pick, float(y))
            train.append(pick)
            f_best = min(f_best, float(y))
            if (t + 1) in check:  # the oracle refits from scratch, like the reference (gp.hpp:81-135)
                model = O.fit(nu, lengthscale, s2, coords[train], values[train], noise, jitter)
            else:
                model = None
        if model is None and (t + 1) in check:
            model = O.fit(nu, lengthscale, s2, coords[train], values[train], noise, jitter)
    run.close()
    return rep
