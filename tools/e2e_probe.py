import sys, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
import paper_2111_14991_b200 as gt
cfg = bench.CONFIGS["c4"]
coords, ids, values = bench.make_workload(cfg)
space = gt.Space(coords)
run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0), n_max=400)
pos = bench.prefix_positions(values, 219, bench.BASE_SEED)
run.fit(pos, values[pos])
for p in pos: run.mark_visited(int(p))
cv = gt.ContextualVarianceState(float(np.mean(values[pos[:20]])), run.mean_variance())
expl = gt.ExplorationConfig(); fb = float(np.min(values[pos]))
af = gt.AcquisitionId.ei
pick = run.select([af], fb, expl, cv).pick(af)
def loop(k, rollback, unmark=True):
    global pick
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k):
        if rollback: run.truncate_async(219)
        _, s = run.observe(pick, float(values[pick]), [af], fb, expl, cv)
        if rollback and unmark: run.unmark_visited(pick)
        pick = s.pick(af)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e6
print("with rollback us/iter", loop(60, True), loop(60, True))
print("truncate only (visited set grows) us/iter", loop(200, True, False), loop(200, True, False))
print("growing model (no rollback, n 220->280) us/iter", loop(60, False))
