"""Device phases of the per-iteration gtc_observe path at the C4 shape
(GTC_PHASE_EVENTS=1: CUDA events around append | pass | selection) next to
the wall clock of the same calls without events.  Diagnostic."""
import os
import pathlib
import sys
import time

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2111_14991_b200 as gt  # noqa: E402

cfg = bench.CONFIGS["c4"]
coords, ids, values = bench.make_workload(cfg)
space = gt.Space(coords)
run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0), n_max=400)
pos = bench.prefix_positions(values, 219, bench.BASE_SEED)
run.fit(pos, values[pos])
for p in pos:
    run.mark_visited(int(p))
cv = gt.ContextualVarianceState(float(np.mean(values[pos[:20]])), run.mean_variance())
expl, fb, af = gt.ExplorationConfig(), float(np.min(values[pos])), gt.AcquisitionId.ei
pick = run.select([af], fb, expl, cv).pick(af)
ph = []
for it in range(60):
    run.truncate_async(219)
    _, s = run.observe(pick, float(values[pick]), [af], fb, expl, cv)
    pick = s.pick(af)
    if os.environ.get("GTC_PHASE_EVENTS"):
        out = (gt._lib.C.c_double * 3)() if hasattr(gt._lib, "C") else None
        import ctypes as C
        out = (C.c_double * 3)()
        gt.load().gtc_last_phase_ms(run.handle, out)
        ph.append([1e3 * x for x in out])
if ph:
    a = np.median(np.array(ph[10:]), axis=0)
    print("median us: append %.2f  pass %.2f  select %.2f  sum %.2f" % (a[0], a[1], a[2], a.sum()))
t0 = time.perf_counter()
for it in range(200):
    run.truncate_async(219)
    _, s = run.observe(pick, float(values[pick]), [af], fb, expl, cv)
    pick = s.pick(af)
print("wall us/iter %.2f" % ((time.perf_counter() - t0) / 200 * 1e6))
