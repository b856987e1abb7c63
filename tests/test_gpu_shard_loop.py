"""Device-resident candidate-axis sharding (gtc_comm + gtc_run_attach_comm +
gtc_run_steps): one BO run's candidates split over shards, the per-iteration
exchanges (selection records, variance accumulators) enqueued on the device.
Every pick, lambda and value must equal the unsharded resident loop's
(strategies.hpp:401-449; the merge applies best_candidate's rule over the
union of the shards, portfolio.hpp:32-61; the variance totals sum exactly).
Shards run on one GPU here (in-process group, one host thread per shard, peer
copies ordered by CUDA events); NCCL is exercised at world size 1."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2111_14991_b200 import synthetic
from paper_2111_14991_b200.sharding import Comm, ShardedRun, split_tiles

pytestmark = pytest.mark.gpu


def workload(gt, grid, invalid, seed, n_init, n_max, nu=1):
    coords, ids, values = synthetic.random_rough(grid, seed, invalid)
    kern = gt.MaternKernel(gt.MaternNu(nu), 1.5, 1.0)
    rng = np.random.default_rng(seed)
    valid = np.nonzero(~np.isnan(values))[0]
    init = rng.choice(valid, n_init, replace=False)
    return coords, values, kern, init


def unsharded(gt, coords, values, kern, init, n_max, af, k, expl, portfolio=None, hold=False):
    space = gt.Space(coords)
    run = gt.SurrogateRun(space, kern, 1e-10, 1e-6, n_max)
    run.fit(init, values[init])
    for p in init:
        run.mark_visited(int(p))
    cv = gt.ContextualVarianceState(float(np.mean(values[init])), run.mean_variance())
    run.set_values(values)
    if portfolio is not None:
        run.set_portfolio(portfolio)
    f0 = float(np.min(values[init]))
    recs = run.steps(af, k, f0, expl, cv, hold=hold)
    out = [(r.position, r.value, r.lambda_, r.valid, r.by) for r in recs]
    m, v = run.predictions()
    run.close()
    space.close()
    return out, cv, m, v


def sharded(gt, coords, values, kern, init, n_max, af, k, expl, cv, parts, portfolio=None, hold=False,
            comms=None, chunks=(None,)):
    N = len(values)
    comms = comms or Comm.local_group(parts)
    shards = []
    for r in range(parts):
        lo, hi = split_tiles(N, parts, r)
        sh = ShardedRun(coords[lo:hi], lo, N, comms[r], kern, 1e-10, 1e-6, n_max)
        sh.fit_points(coords[init], values[init])
        for p in init:
            sh.mark_global(int(p))
        sh.set_values(values)
        if portfolio is not None:
            sh.run.set_portfolio(portfolio)
        shards.append(sh)
    f0 = float(np.min(values[init]))

    def drive(sh):
        out = []
        fb = f0
        for c in chunks:
            recs = sh.steps(af, c or k, fb, expl, cv, hold=hold)
            out += [(r.position, r.value, r.lambda_, r.valid, r.by) for r in recs]
            vs = [r.value for r in recs if r.valid]
            if vs and not hold:
                fb = min(fb, min(vs))
        return out

    with ThreadPoolExecutor(parts) as ex:
        results = list(ex.map(drive, shards))
    preds = [sh.run.predictions() for sh in shards]
    m = np.concatenate([p[0] for p in preds])
    v = np.concatenate([p[1] for p in preds])
    for sh in shards:
        sh.close()
    for c in comms:
        c.close()
    return results, m, v


def same(a, b):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert x[0] == y[0] and x[3] == y[3] and x[4] == y[4]
        assert (np.isnan(x[1]) and np.isnan(y[1])) or x[1] == y[1]
        assert x[2] == y[2]  # lambda bit for bit (exact fixed-point totals)


@pytest.mark.parametrize("parts", [2, 3])
@pytest.mark.parametrize("af,invalid", [(0, 0.0), (2, 0.3), (1, 0.1)])
def test_sharded_steps_equal_unsharded(gt, parts, af, invalid):
    af = gt.AcquisitionId(af)
    expl = gt.ExplorationConfig()
    coords, values, kern, init = workload(gt, [10, 10, 10, 8, 6], invalid, 31 + int(af), 20, 220)
    ref, cv, m_ref, v_ref = unsharded(gt, coords, values, kern, init, 220, af, 200, expl)
    res, m, v = sharded(gt, coords, values, kern, init, 220, af, 200, expl, cv, parts)
    for out in res:  # every shard reports the same global trajectory
        same(out, ref)
    assert len(ref) == 200
    if invalid > 0:
        assert any(not r[3] for r in ref)
    # the posterior over the union of the shards is the unsharded one
    np.testing.assert_array_equal(m, m_ref[:len(m)])
    np.testing.assert_array_equal(v, v_ref[:len(v)])


def test_sharded_steps_chunked_constant_lambda(gt):
    """Several gtc_run_steps calls in a row (host bookkeeping replayed from
    the records' coordinates between chunks), constant lambda, nu = 5/2."""
    af = gt.AcquisitionId.ei
    expl = gt.ExplorationConfig(gt.ExplorationConfig.Mode.constant, 0.01)
    coords, values, kern, init = workload(gt, [9, 9, 9, 9, 4], 0.2, 77, 15, 160, nu=2)
    ref, cv, _, _ = unsharded(gt, coords, values, kern, init, 160, af, 120, expl)
    res, _, _ = sharded(gt, coords, values, kern, init, 160, af, 120, expl, cv, 2, chunks=(40, 40, 40))
    for out in res:
        same(out, ref)


def test_sharded_portfolio_multi(gt):
    """bo-multi on the device portfolio (all three AF winners shipped per shard)."""
    coords, values, kern, init = workload(gt, [10, 10, 10, 10, 3], 0.25, 5, 20, 200)
    expl = gt.ExplorationConfig()
    pc = 1  # GTC_PORTFOLIO_MULTI
    af = gt.AcquisitionId.ei
    ref, cv, _, _ = unsharded(gt, coords, values, kern, init, 200, af, 150, expl, portfolio=pc)
    res, _, _ = sharded(gt, coords, values, kern, init, 200, af, 150, expl, cv, 3, portfolio=pc)
    assert len({r[4] for r in ref}) > 1  # several functions picked
    for out in res:
        same(out, ref)


def test_sharded_hold_c4(gt):
    """The bench's steady state (BASELINE configs[3]): C4, N = 1M, n = 220,
    bo-ei, contextual variance, hold mode; 2 shards on one device."""
    import bench
    coords, ids, values = bench.make_workload(bench.CONFIGS["c4"])
    kern = gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0)
    init = bench.prefix_positions(values, 219, bench.BASE_SEED)
    af = gt.AcquisitionId.ei
    expl = gt.ExplorationConfig()
    ref, cv, _, _ = unsharded(gt, coords, values, kern, init, 220, af, 40, expl, hold=True)
    res, _, _ = sharded(gt, coords, values, kern, init, 220, af, 40, expl, cv, 2, hold=True)
    for out in res:
        same(out, ref)


def test_nccl_world1(gt):
    """The NCCL transport at world size 1 (ncclAllGather on the run's stream)."""
    try:
        uid = Comm.nccl_unique_id()
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"NCCL unavailable: {e}")
    comm = Comm.nccl(uid, 0, 1, 0)
    assert comm.size == 1 and comm.rank == 0
    af = gt.AcquisitionId.lcb
    expl = gt.ExplorationConfig()
    coords, values, kern, init = workload(gt, [10, 10, 10, 10, 2], 0.3, 9, 20, 200)
    ref, cv, _, _ = unsharded(gt, coords, values, kern, init, 200, af, 150, expl)
    res, _, _ = sharded(gt, coords, values, kern, init, 200, af, 150, expl, cv, 1, comms=[comm])
    same(res[0], ref)


def test_attach_rejects_unaligned_offset(gt):
    comms = Comm.local_group(2)
    coords, values, kern, init = workload(gt, [8, 8, 8], 0.0, 1, 5, 20)
    with pytest.raises(gt.Error, match="multiple of 256"):
        ShardedRun(coords[100:], 100, len(values), comms[1], kern, n_max=20)
    for c in comms:
        c.close()
