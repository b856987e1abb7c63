"""Distribution of the EI standardised margin z = (best - lambda - mu)/sd over
the C4 bench state (how much of the candidate set the pruned selection can
discard).  Diagnostic only."""
import sys

import numpy as np

sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import paper_2111_14991_b200 as gt  # noqa: E402
from paper_2111_14991_b200 import synthetic  # noqa: E402
from paper_2111_14991_b200 import AcquisitionId, ContextualVarianceState, ExplorationConfig  # noqa: E402

coords, ids, values = synthetic.random_rough([10] * 6, 20261017, 0.0)
space = gt.Space(coords)
run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0), n_max=220)
rng = np.random.default_rng(20261017)
pos = rng.choice(len(values), 219, replace=False)
y = values[pos]
run.fit(pos, y)
for p in pos:
    run.mark_visited(int(p))
cv = ContextualVarianceState(float(np.mean(y[:20])), run.mean_variance())
for af in (AcquisitionId.ei, AcquisitionId.poi, AcquisitionId.lcb):
    sel = run.select([af], float(np.min(y)), ExplorationConfig(), cv)
    mu, var = run.predictions()
    mask = np.ones(len(mu), bool)
    mask[pos] = False
    sd = np.sqrt(var[mask])
    lam, best = sel.lambda_, sel.best_std
    z = (best - lam - mu[mask]) / sd if af == AcquisitionId.ei else (best + lam - mu[mask]) / sd
    print(af.name, "lambda", lam, "best_std", best, "pick", sel.pick(af), "score", sel.score[int(af)])
    print("  z quantiles", np.quantile(z, [0, 0.001, 0.01, 0.1, 0.5, 0.9, 0.99, 0.999, 1]))
    print("  sd quantiles", np.quantile(sd, [0, 0.01, 0.5, 0.99, 1]))
    s = gt.acquisition_scores(af, mu[mask], sd, best, lam)
    top = np.max(s)
    for f in (0.5, 0.9, 0.99, 0.999):
        print(f"  candidates with score >= {f} * max: {np.sum(s >= f * top) if top > 0 else np.sum(s >= top / f)}")
