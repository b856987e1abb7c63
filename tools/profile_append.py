import sys, numpy as np, ctypes as C
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import paper_2111_14991_b200 as gt
from paper_2111_14991_b200 import synthetic, _lib
coords, ids, values = synthetic.random_rough([10]*6, 20261017, 0.0)
space = gt.Space(coords)
run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.three_halves, 1.5), n_max=220)
rng = np.random.default_rng(1); pos = rng.choice(len(values), 220, replace=False)
run.fit(pos[:219], values[pos[:219]])
cv = gt.ContextualVarianceState(float(np.mean(values[pos[:20]])), run.mean_variance())
for it in range(5):
    run.truncate_async(219)
    run.observe(int(pos[219]), float(values[pos[219]]), [gt.AcquisitionId.ei], 1.0, gt.ExplorationConfig(), cv)
    run.unmark_visited(int(pos[219]))
    m = (C.c_uint64 * 7)()
    gt.load().gtc_debug_append_marks(run.handle, m)
    t = np.array(list(m), dtype=np.int64)
    print("append phases us:", np.round(np.diff(t) / 1e3, 2), "total", (t[6]-t[0])/1e3, "step ms", run.last_step_ms(), "pass ms", run.last_pass_ms())
