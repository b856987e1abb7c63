"""Candidate-axis sharding protocol on one device: a space split into shards
(each its own resident space + replicated GP, observations applied with
explicit coordinates) must pick the same configurations as the unsharded run
and agree on lambda to rounding (the global variance sum is reduced per shard,
then in rank order)."""
import numpy as np
import pytest

from paper_2111_14991_b200 import synthetic
from paper_2111_14991_b200.sharding import Shard, ShardGroup, split_bounds

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("parts,afs", [(2, (0,)), (3, (0, 1, 2)), (4, (2,))])
def test_sharded_loop_matches_unsharded(gt, parts, afs):
    coords, ids, values = synthetic.random_rough([12, 10, 9, 8], 5, 0.0)
    N = len(values)
    kern = gt.MaternKernel(gt.MaternNu.three_halves, 1.5)
    afs = [gt.AcquisitionId(a) for a in afs]
    rng = np.random.default_rng(parts)
    init = rng.choice(N, 12, replace=False)
    y0 = values[init]

    full = gt.SurrogateRun(gt.Space(coords), kern, n_max=64)
    full.fit(init, y0)
    for p in init:
        full.mark_visited(int(p))

    shards = []
    for r in range(parts):
        lo, hi = split_bounds(N, parts, r)
        sh = Shard(coords[lo:hi], lo, kern, n_max=64)
        sh.fit_points(coords[init], y0)
        for p in init:
            sh.mark_global(int(p))
        shards.append(sh)
    group = ShardGroup(shards)

    cv = gt.ContextualVarianceState(float(np.mean(y0)), full.mean_variance())
    assert group.mean_variance() == pytest.approx(cv.initial_mean_variance, rel=1e-13)
    expl = gt.ExplorationConfig()
    fb = float(np.min(y0))
    s_full = full.select(afs, fb, expl, cv)
    s_shard = group.select(afs, fb, expl, cv)
    for it in range(25):
        assert s_shard.position == s_full.position, it
        assert s_shard.n_candidates == s_full.n_candidates
        assert s_shard.lambda_ == pytest.approx(s_full.lambda_, rel=1e-12)
        pick = s_full.position[int(afs[it % len(afs)])]
        y = float(values[pick])
        fb = min(fb, y)
        _, s_full = full.observe(pick, y, afs, fb, expl, cv)
        s_shard = group.observe(coords[pick], pick, y, afs, fb, expl, cv)


def test_sharded_invalid_observation_and_exclusion(gt):
    coords, ids, values = synthetic.random_rough([20, 20], 3, 0.0)
    N = len(values)
    kern = gt.MaternKernel()
    init = np.array([5, 77, 203, 311])
    shards = [Shard(coords[lo:hi], lo, kern, n_max=16) for lo, hi in (split_bounds(N, 2, r) for r in range(2))]
    for sh in shards:
        sh.fit_points(coords[init], values[init])
        for p in init:
            sh.mark_global(int(p))
    group = ShardGroup(shards)
    sel = group.select([gt.AcquisitionId.ei], 1.0, gt.ExplorationConfig(gt.ExplorationConfig.Mode.constant))
    p = sel.position[0]
    sel2 = group.select([gt.AcquisitionId.ei], 1.0, gt.ExplorationConfig(gt.ExplorationConfig.Mode.constant),
                        excluded=[p])
    assert sel2.position[0] != p and sel2.n_candidates == sel.n_candidates - 1
    # an invalid observation marks visited on the owner only, model unchanged
    sel3 = group.observe(coords[p], p, None, [gt.AcquisitionId.ei], 1.0,
                         gt.ExplorationConfig(gt.ExplorationConfig.Mode.constant))
    assert sel3.position[0] == sel2.position[0] and sel3.n_candidates == sel.n_candidates - 1
