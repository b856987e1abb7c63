"""Exactness of the pruned selection (gtc_kernels.cu select_pruned).

The device argmax scores exactly only the candidates whose FP32 upper bound
reaches the block's threshold.  These tests compare it with the argmax of the
FULL score array computed on the device by the same FP64 formulas
(gtc_acquisition_scores), with the reference's rule (portfolio.hpp:32-61:
higher score, then lower position; NaN scores skipped; the first candidate is
taken unconditionally), so any pruning error shows up as a different position,
bit for bit.  The inputs are built to stress the bounds: PI saturation at 1.0,
EI deep in the tail (z << -13, subnormal scores), exact ties spread across
blocks, sd == 0, NaN/inf/huge values, sizes that are not chunk multiples and
more candidates than one wave of blocks.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def full_argmax(gt, af, means, stds, best, lam, excluded=None):
    s = gt.acquisition_scores(gt.AcquisitionId(af), means, stds, best, lam)
    elig = np.ones(len(s), bool) if excluded is None else ~np.asarray(excluded, bool)
    idx = np.nonzero(elig)[0]
    first = idx[0]
    if np.isnan(s[first]):
        return first
    cand = idx[~np.isnan(s[idx])]
    top = s[cand].max()
    return int(cand[np.nonzero(s[cand] == top)[0][0]])


def check(gt, af, means, stds, best, lam, excluded=None):
    c = gt.CandidateScores(np.arange(len(means)), means, stds, best, lam)
    got = gt.best_candidate(gt.AcquisitionId(af), c, excluded)
    want = full_argmax(gt, af, means, stds, best, lam, excluded)
    assert got == want, (af, got, want)
    return got


@pytest.mark.parametrize("af", [0, 1, 2])
@pytest.mark.parametrize("n", [1, 7, 513, 70_001, 1_000_000, 1_700_000])
def test_random_landscapes(gt, af, n):
    rng = np.random.default_rng(100 + n + af)
    means = rng.normal(size=n)
    stds = rng.random(n)
    for best, lam in ((-1.5, 0.01), (0.0, 0.3), (-4.0, 0.0)):
        check(gt, af, means, stds, best, lam)


@pytest.mark.parametrize("af", [0, 1, 2])
def test_planted_exact_ties_across_blocks(gt, af):
    """The maximum value appears at many positions in different blocks: the
    lowest position must win even when it sits in a later chunk."""
    rng = np.random.default_rng(5)
    n = 1_300_000
    means = 1.0 + rng.random(n)
    stds = 0.2 * rng.random(n)
    top = rng.choice(n, 40, replace=False)
    means[top] = -2.0
    stds[top] = 0.9
    got = check(gt, af, means, stds, -1.0, 0.05)
    assert got == top.min()


def test_pi_saturation(gt):
    """Half the candidates have PI == 1.0 exactly (z > 8.3): the lowest of them."""
    rng = np.random.default_rng(11)
    n = 600_000
    means = rng.normal(size=n)
    stds = 0.05 + rng.random(n)
    sat = rng.random(n) < 0.5
    means[sat] = -50.0
    stds[sat] = 1.0
    got = check(gt, 1, means, stds, 0.0, 0.01)
    assert got == np.nonzero(sat)[0][0]


@pytest.mark.parametrize("af", [0, 1])
def test_deep_tail_scores(gt, af):
    """Every candidate has z in [-40, -14]: EI/PI are tiny or subnormal (beyond
    the FP32 bound range), so the caps must keep the exact argmax."""
    rng = np.random.default_rng(12)
    n = 400_000
    stds = 0.01 + 0.02 * rng.random(n)
    z = -14.0 - 26.0 * rng.random(n)
    means = -z * stds
    check(gt, af, means, stds, 0.0, 0.0)


@pytest.mark.parametrize("af", [0, 1, 2])
def test_nonfinite_and_degenerate_inputs(gt, af):
    rng = np.random.default_rng(13)
    n = 300_000
    means = rng.normal(size=n)
    stds = rng.random(n)
    k = rng.choice(n, 600, replace=False)
    means[k[:100]] = np.nan
    stds[k[100:200]] = np.nan
    stds[k[200:300]] = 0.0
    means[k[300:400]] = 1e31
    means[k[400:450]] = -1e31
    stds[k[450:500]] = 1e20
    stds[k[500:550]] = np.inf
    stds[k[550:600]] = 1e-20
    excluded = (rng.random(n) < 0.1).astype(np.uint8)
    excluded[: k.min()] = 1  # the first eligible candidate is a degenerate one
    for best, lam in ((-0.5, 0.1), (0.0, 0.0)):
        check(gt, af, means, stds, best, lam, excluded)


@pytest.mark.parametrize("af", [0, 1, 2])
def test_first_candidate_nan_rule(gt, af):
    n = 200_000
    rng = np.random.default_rng(14)
    means = rng.normal(size=n)
    stds = rng.random(n)
    means[0] = np.nan
    assert check(gt, af, means, stds, -1.0, 0.1) == 0
    excluded = np.zeros(n, np.uint8)
    excluded[:1000] = 1
    means[1000] = np.nan
    assert check(gt, af, means, stds, -1.0, 0.1, excluded) == 1000


@pytest.mark.parametrize("af", [0, 1, 2])
def test_near_equal_landscape(gt, af):
    """Scores that differ in the last few ulps (quantised means, constant sd):
    every candidate's bound passes the threshold, exact scoring decides."""
    rng = np.random.default_rng(15)
    n = 500_000
    means = 0.3 + np.round(rng.random(n), 2) * 1e-13
    stds = np.full(n, 0.25)
    check(gt, af, means, stds, 0.2, 0.01)
