"""One GP fit (factorisation + full V rebuild + posterior) at the C4 shape
(N = 1M, d = 6, n = 220), timed on the host around synchronised calls; run
under `ncu --metrics gpu__time_duration.sum` for the per-kernel split.
Diagnostic only."""
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2111_14991_b200 as gt  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 220
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
coords, ids, values = bench.make_workload(bench.CONFIGS["c4"])
space = gt.Space(coords)
run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0), n_max=n)
pos = bench.prefix_positions(values, n, bench.BASE_SEED)
y = values[pos]
ts = []
for r in range(reps):
    t0 = time.perf_counter()
    run.fit(pos, y)
    m, v = run.predictions()  # (synchronises)
    ts.append(1e3 * (time.perf_counter() - t0))
print({"n": n, "fit_ms": [round(t, 3) for t in ts]})
