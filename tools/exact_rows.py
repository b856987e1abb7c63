"""How often the resident loop's bordered row needs the exact substitution
(V-column pivot below the 2^-8 margin): BO runs of 220 evaluations on the
BASELINE case spaces and the golden trajectory spaces.  Diagnostic.

  python tools/exact_rows.py
"""
import json
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2111_14991_b200 as gt  # noqa: E402

out = []
for path in sorted((ROOT / "tests" / "golden").glob("case_*.npz")) + sorted((ROOT / "tests" / "golden").glob("traj_*.npz")):
    t = np.load(path)
    if "coords" in t:
        space, values = gt.Space(t["coords"]), t["values"]
    elif "spec" in t:
        spec = json.loads(str(t["spec"]))
        es = gt.SearchSpace([gt.ParameterDef(p["name"], p["values"]) for p in spec["params"]],
                            spec["restrictions"]).enumerate()
        space, values = es, t["values"]
    else:
        continue
    for nu in (gt.MaternNu.three_halves,):
        run = gt.SurrogateRun(space, gt.MaternKernel(nu, 1.5, 1.0), n_max=230)
        rng = np.random.default_rng(1)
        valid = np.flatnonzero(~np.isnan(values))
        pos = rng.choice(valid, 10, replace=False)
        run.fit(pos, values[pos])
        for p in pos:
            run.mark_visited(int(p))
        run.set_values(values)
        cv = gt.ContextualVarianceState(float(np.mean(values[pos])), run.mean_variance())
        recs = run.steps(gt.AcquisitionId.ei, 210, float(np.min(values[pos])), gt.ExplorationConfig(), cv)
        nvalid = sum(1 for r in recs if r.valid)
        out.append({"case": path.stem, "N": int(space.n), "steps": len(recs), "valid": nvalid,
                    "exact_rows": run.exact_rows()})
        print(out[-1], flush=True)
