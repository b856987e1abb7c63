"""The full factorisation and V rebuild of GpModel::fit on the device.

The right-looking shared-memory factor (k_gp_factor_rl) against the
left-looking bordered rows (k_gp_factor), and the tensor-core V rebuild (k_rebuild: FP64 mma.sync panels, one pass) against
the streaming rebuild (k_extend<8>, n/8 passes) -- the full forward
substitution of GpModel::predict (gp.hpp:150-168) that fits, refits and the
stand-alone predict run.  The DMMA chain is an ascending FMA chain, so the two
must agree BIT FOR BIT: posterior mean/variance, the variance total (lambda's
input) and every later incremental append (which reads the rebuilt V rows)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture
def rebuild_mode(gt):
    lib = gt.load()
    prev = lib.gtc_debug_set_rebuild(-1)
    yield lambda m: lib.gtc_debug_set_rebuild(m)
    lib.gtc_debug_set_rebuild(prev)


def fitted(gt, coords, nu, pos, y, mode, set_mode, extra=None):
    set_mode(mode)
    space = gt.Space(coords)
    run = gt.SurrogateRun(space, gt.MaternKernel(nu, 1.3, 0.9), n_max=len(pos) + 2)
    run.fit(pos, y)
    mu, var = run.predictions()
    out = [mu.copy(), var.copy(), run.mean_variance()]
    if extra is not None:  # one incremental append on top of the rebuilt rows
        run.append(int(extra[0]), float(extra[1]))
        mu2, var2 = run.predictions()
        out += [mu2.copy(), var2.copy()]
    return out


@pytest.mark.parametrize("mode", [1, 2, 3, 4])
@pytest.mark.parametrize("nu", ["half", "three_halves", "five_halves"])
@pytest.mark.parametrize("n", [1, 7, 8, 9, 37, 64, 150])
def test_rebuild_bit_identical_to_streaming(gt, rebuild_mode, nu, n, mode):
    rng = np.random.default_rng(n * 7 + len(nu))
    N, d = 20_000 + 37 * n, 5
    grid = np.linspace(0.0, 1.0, 11)
    coords = grid[rng.integers(0, 11, size=(N, d))]  # discrete: the compact 1-byte coordinate path
    pos = rng.choice(N, n + 1, replace=False)
    y = 2.0 + rng.standard_normal(n + 1)
    mnu = getattr(gt.MaternNu, nu)
    a = fitted(gt, coords, mnu, pos[:n], y[:n], 0, rebuild_mode, extra=(pos[n], y[n]))
    b = fitted(gt, coords, mnu, pos[:n], y[:n], mode, rebuild_mode, extra=(pos[n], y[n]))
    for x, z in zip(a, b):
        np.testing.assert_array_equal(np.asarray(x), np.asarray(z))


@pytest.mark.parametrize("mode", [1, 2, 3, 4])
def test_rebuild_continuous_coordinates_and_n220(gt, rebuild_mode, mode):
    """Non-discrete coordinates (the FP64 SoA path) at the headline n = 220."""
    rng = np.random.default_rng(5)
    N, d, n = 60_000, 6, 220
    coords = rng.random((N, d))
    pos = rng.choice(N, n, replace=False)
    y = rng.standard_normal(n)
    a = fitted(gt, coords, gt.MaternNu.three_halves, pos, y, 0, rebuild_mode)
    b = fitted(gt, coords, gt.MaternNu.three_halves, pos, y, mode, rebuild_mode)
    for x, z in zip(a, b):
        np.testing.assert_array_equal(np.asarray(x), np.asarray(z))


@pytest.mark.parametrize("n", [300, 420])
def test_rebuild_large_n_persistent_passes_and_fallback(gt, rebuild_mode, n):
    """Mode 4 (persistent 64-row DMMA passes) at n = 300 (five passes, the
    last one partial) and n = 420 (rows of L past its shared-memory budget:
    the 32-row passes take over) -- bit for bit the streaming rebuild."""
    rng = np.random.default_rng(n)
    N, d = 9_000, 4
    grid = np.linspace(0.0, 1.0, 13)
    coords = grid[rng.integers(0, 13, size=(N, d))]
    pos = rng.choice(N, n + 1, replace=False)
    y = rng.standard_normal(n + 1)
    a = fitted(gt, coords, gt.MaternNu.five_halves, pos[:n], y[:n], 0, rebuild_mode, extra=(pos[n], y[n]))
    b = fitted(gt, coords, gt.MaternNu.five_halves, pos[:n], y[:n], 4, rebuild_mode, extra=(pos[n], y[n]))
    for x, z in zip(a, b):
        np.testing.assert_array_equal(np.asarray(x), np.asarray(z))


@pytest.mark.parametrize("mode", [2, 4])
def test_rebuild_high_dimension(gt, rebuild_mode, mode):
    """d = 11 > 8: the kernel values take k_kstar's per-row coordinate path
    (no register copy, norms from global memory) -- still bit for bit."""
    rng = np.random.default_rng(11)
    N, d, n = 12_000, 11, 90
    coords = rng.random((N, d))
    pos = rng.choice(N, n + 1, replace=False)
    y = rng.standard_normal(n + 1)
    a = fitted(gt, coords, gt.MaternNu.five_halves, pos[:n], y[:n], 0, rebuild_mode, extra=(pos[n], y[n]))
    b = fitted(gt, coords, gt.MaternNu.five_halves, pos[:n], y[:n], mode, rebuild_mode, extra=(pos[n], y[n]))
    for x, z in zip(a, b):
        np.testing.assert_array_equal(np.asarray(x), np.asarray(z))


@pytest.fixture
def factor_mode(gt):
    lib = gt.load()
    prev = lib.gtc_debug_set_factor(-1)
    yield lambda m: lib.gtc_debug_set_factor(m)
    lib.gtc_debug_set_factor(prev)


@pytest.mark.parametrize("nu", ["half", "three_halves", "five_halves"])
@pytest.mark.parametrize("n", [1, 2, 33, 100, 220])
def test_right_looking_factor_bit_identical(gt, factor_mode, nu, n):
    """Same factor bit for bit: identical posterior, standardisation, fit
    info (jitter) and a later append on top of it."""
    rng = np.random.default_rng(100 + n)
    N, d = 30_000, 4
    coords = rng.random((N, d))
    pos = rng.choice(N, n + 1, replace=False)
    y = rng.standard_normal(n + 1) * 3.0
    out = []
    for mode in (0, 1):
        factor_mode(mode)
        run = gt.SurrogateRun(gt.Space(coords), gt.MaternKernel(getattr(gt.MaternNu, nu), 0.8, 1.1), n_max=n + 2)
        info = run.fit(pos[:n], y[:n])
        mu, var = run.predictions()
        run.append(int(pos[n]), float(y[n]))
        mu2, var2 = run.predictions()
        out.append([mu.copy(), var.copy(), mu2.copy(), var2.copy(), info.jitter, info.y_mean, info.y_std])
    for x, z in zip(*out):
        np.testing.assert_array_equal(np.asarray(x), np.asarray(z))


def test_right_looking_factor_escalates_like_left_looking(gt, factor_mode):
    """Near-duplicate training points at jitter 1e-17 (test_gpu_run's
    escalation case, scaled up): the same failing pivot, the same escalated
    jitter, the same posterior from both factorisations."""
    rng = np.random.default_rng(9)
    coords = rng.random((3_000, 2))
    coords[1] = coords[0] + np.array([1e-9, 0.0])
    coords[11] = coords[10] + np.array([0.0, 1e-9])
    pos = np.concatenate([[0, 1, 10, 11], rng.choice(np.arange(20, 3_000), 40, replace=False)])
    y = rng.standard_normal(len(pos))
    out = []
    for mode in (0, 1):
        factor_mode(mode)
        run = gt.SurrogateRun(gt.Space(coords), gt.MaternKernel(), 0.0, 1e-17, len(pos) + 1)
        info = run.fit(pos, y)
        mu, var = run.predictions()
        out.append([mu.copy(), var.copy(), info.jitter])
    assert out[0][2] > 1e-17  # the escalation happened
    for x, z in zip(*out):
        np.testing.assert_array_equal(np.asarray(x), np.asarray(z))
