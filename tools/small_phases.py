"""Diagnostics: per-iteration phases of the resident loop on small spaces
(hold mode at n = 220): selection (+ loop advance), bordered append, pass."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_14991_b200 as gt  # noqa: E402
from paper_2111_14991_b200 import synthetic  # noqa: E402

for grid in ([12, 8, 8, 12], [10, 10, 10, 10, 10], [10, 10, 10, 10, 5, 2]):
    coords, ids, values = synthetic.random_rough(grid, 5, 0.0)
    space = gt.Space(coords)
    run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0), n_max=220)
    rng = np.random.default_rng(1)
    pos = rng.choice(len(values), 219, replace=False)
    run.fit(pos, values[pos])
    for p in pos:
        run.mark_visited(int(p))
    cv = gt.ContextualVarianceState(float(np.mean(values[pos[:20]])), run.mean_variance())
    run.set_values(values)
    fb = float(np.min(values[pos]))
    run.steps(gt.AcquisitionId.ei, 20, fb, gt.ExplorationConfig(), cv, hold=True)
    run.truncate_async(219)
    run.steps(gt.AcquisitionId.ei, 100, fb, gt.ExplorationConfig(), cv, hold=True, timing=True)
    ph = run.last_steps_phase_ms()
    run.truncate_async(219)
    run.steps(gt.AcquisitionId.ei, 100, fb, gt.ExplorationConfig(), cv, hold=True)
    print(f"N={len(values)}: selection {1e3 * ph[0]:.1f} append {1e3 * ph[1]:.1f} pass {1e3 * ph[2]:.1f} us; "
          f"chunk {1e3 * run.last_steps_ms() / 100:.1f} us/iteration (PDL, no events)", flush=True)
