"""Acquisition + masked argmax on the device (port of
/root/reference/proj/tests/test_acquisition.cpp and test_portfolio.cpp's
best_candidate cases), through gtc_acquisition_scores / gtc_best_candidate."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def score1(gt, af, mean, std, best, lam):
    return float(gt.acquisition_scores(af, [mean], [std], best, lam)[0])


def test_pi_closed_form(gt):  # test_acquisition.cpp:15-23
    A = gt.AcquisitionId
    assert score1(gt, A.poi, 1.3, 1.0, 1.2, 0.1) == 0.5
    assert score1(gt, A.poi, 2.0, 0.0, 1.0, 0.5) == 0.0
    assert score1(gt, A.poi, 0.5, 0.0, 1.0, 0.5) == 1.0
    assert abs(score1(gt, A.poi, 1.0 + 0.2 - 1.96 * 0.7, 0.7, 1.0, 0.2) - 0.9750021048517795) <= 1e-9


def test_ei_closed_form(gt):  # test_acquisition.cpp:25-32
    A = gt.AcquisitionId
    assert score1(gt, A.ei, 1.0, 0.0, 1.0, 0.0) == 0.0
    assert score1(gt, A.ei, 2.0, 0.0, 1.5, 0.3) == 0.0
    assert score1(gt, A.ei, 1.0, 0.0, 2.0, 0.5) == 0.5
    assert abs(score1(gt, A.ei, 1.0, 1.0, 1.0, 0.0) - 0.3989422804014327) <= 1e-12


def test_lcb_direct_arithmetic(gt):  # test_acquisition.cpp:59-63 (score = -lcb)
    A = gt.AcquisitionId
    assert score1(gt, A.lcb, 1.0, 0.5, 0.0, 2.0) == -0.0
    assert score1(gt, A.lcb, 1.7, 3.0, 0.0, 0.0) == -1.7
    assert score1(gt, A.lcb, 1.7, 0.0, 0.0, 5.0) == -1.7


def test_scores_match_oracle_and_invariants(gt, oracle):
    """test_acquisition.cpp:65-79 invariants on 20k draws, plus per-value
    parity with the oracle at 1e-12 relative (1e-9 is the contract)."""
    rng = np.random.default_rng(9)
    n = 20_000
    mean = -3.0 + 6.0 * rng.random(n)
    std = 2.0 * rng.random(n)
    std[:50] = 0.0
    best, lam = 0.37, 0.61
    ei = gt.acquisition_scores(gt.AcquisitionId.ei, mean, std, best, lam)
    pi = gt.acquisition_scores(gt.AcquisitionId.poi, mean, std, best, lam)
    nl = gt.acquisition_scores(gt.AcquisitionId.lcb, mean, std, best, lam)
    assert np.all(ei >= 0) and np.all(pi >= 0) and np.all(pi <= 1) and np.all(-nl <= mean + 1e-15)
    for i in range(0, n, 97):
        assert abs(ei[i] - oracle.ei(mean[i], std[i], best, lam)) <= 1e-12 * max(1.0, abs(ei[i]))
        assert abs(pi[i] - oracle.pi(mean[i], std[i], best, lam)) <= 1e-12
        assert nl[i] == -oracle.lcb(mean[i], std[i], lam)
    assert score1(gt, gt.AcquisitionId.ei, 1.5, 0.4, 1.0, 0.0) > 0.0


def cs(gt, means, stds, best=0.0, lam=0.0):
    return gt.CandidateScores(np.arange(len(means)), np.asarray(means, float), np.asarray(stds, float), best, lam)


def test_ties_resolve_to_lowest_index(gt):  # test_portfolio.cpp:21-29
    for af in gt.AcquisitionId:
        assert gt.best_candidate(af, cs(gt, [0.5] * 3, [1.0] * 3)) == 0


def test_respects_exclusions(gt):  # test_portfolio.cpp:31-40
    c = cs(gt, [-5.0, 0.0, 1.0], [1.0] * 3)
    assert gt.best_candidate(gt.AcquisitionId.ei, c, [True, False, False]) == 1
    with pytest.raises(gt.Error, match="no candidates remaining"):
        gt.best_candidate(gt.AcquisitionId.ei, c, [True, True, True])


def test_crafted_disagreement(gt):  # test_portfolio.cpp:61-71
    c = cs(gt, [0.0, -2.5, -0.5], [0.1, 0.5, 1.2], 0.0, 3.0)
    assert gt.best_candidate(gt.AcquisitionId.poi, c) == 0
    assert gt.best_candidate(gt.AcquisitionId.ei, c) == 1
    assert gt.best_candidate(gt.AcquisitionId.lcb, c) == 2


def test_first_candidate_rule_with_nan(gt):  # portfolio.hpp:52 semantics
    assert gt.best_candidate(gt.AcquisitionId.lcb, cs(gt, [np.nan, -1.0], [1.0, 1.0])) == 0
    assert gt.best_candidate(gt.AcquisitionId.lcb, cs(gt, [1.0, np.nan, -1.0], [1.0] * 3)) == 2
    assert gt.best_candidate(gt.AcquisitionId.lcb, cs(gt, [0.0, np.nan, -1.0], [1.0] * 3), [1, 0, 0]) == 1


@pytest.mark.parametrize("af", [0, 1, 2])
def test_large_argmax_matches_oracle(gt, oracle, af):
    """1M candidates with ties planted: device argmax == oracle argmax (same
    inputs), exclusions honoured."""
    rng = np.random.default_rng(af)
    n = 1_000_000
    means = np.round(rng.normal(size=n), 3)
    stds = np.round(rng.random(n), 3)
    excluded = (rng.random(n) < 0.2).astype(np.uint8)
    best, lam = -1.2, 0.3
    c = gt.CandidateScores(np.arange(n), means, stds, best, lam)
    got = gt.best_candidate(gt.AcquisitionId(af), c, excluded)
    want, want_score = oracle.best_candidate(af, means, stds, best, lam, excluded)
    if got != want:  # only allowed on an ulp-level near-tie of the libm functions
        s = gt.acquisition_scores(gt.AcquisitionId(af), means[[got, want]], stds[[got, want]], best, lam)
        assert abs(s[0] - s[1]) <= 1e-14 * max(1.0, abs(s[1])), (got, want, s)
    assert not excluded[got]
