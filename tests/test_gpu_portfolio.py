"""The device portfolio of the resident loop (gtc_run_steps for bo-multi /
bo-advanced-multi) against the reference's own Portfolio scenarios
(test_portfolio.cpp:63-240, portfolio.hpp:65-316), driven by explicit scripts
through gtc_portfolio_trace: the same device functions the loop runs."""
import ctypes as C

import pytest

from paper_2111_14991_b200 import _lib

pytestmark = pytest.mark.gpu

EI, POI, LCB = 0, 1, 2
MULTI, ADVANCED = 1, 2


def suggest(picks):
    return (0, -1, list(picks), 0.0)


def record(af, value):
    return (1, af, [0, 0, 0], float(value))


def trace(gt, mode, ops, skip=5, discount=None, rho=0.1, active=None):
    cfg = _lib.gtc_portfolio_config(mode, skip, discount if discount else (0.65 if mode == MULTI else 0.75), rho)
    arr = (_lib.gtc_portfolio_op * len(ops))()
    for i, (kind, af, picks, value) in enumerate(ops):
        arr[i].kind, arr[i].af, arr[i].value = kind, af, value
        for a in range(3):
            arr[i].picks[a] = picks[a]
    out = (_lib.gtc_portfolio_state * len(ops))()
    act = (C.c_int32 * 3)(*active) if active is not None else None
    rc = gt.load().gtc_portfolio_trace(0, C.byref(cfg), act, len(ops), arr, out)
    assert rc == 0, _lib.last_error()
    return list(out)


def dos_of(values, gamma):
    d = 0.0
    for v in values:
        d = d * gamma + v
    return d


def test_round_robin_in_fixed_order(gt):
    """test_portfolio.cpp:63-92: PI prefers A (0), EI B (1), LCB C (2); the
    consulted function rotates ei, poi, lcb and no duplicates arise."""
    expected = [EI, POI, LCB, EI, POI, LCB]
    ops = []
    for by in expected:
        ops += [suggest([1, 0, 2]), record(by, 1.0)]
    out = trace(gt, MULTI, ops)
    sug = out[0::2]
    assert [s.by for s in sug] == expected
    assert [s.position for s in sug] == [1, 0, 2, 1, 0, 2]
    assert list(out[-1].active) == [1, 1, 1]
    assert out[-1].duplicates[EI] == 0


def test_multi_skip_after_threshold_keeps_lowest_dos(gt):
    """test_portfolio.cpp:96-130: order (ei, poi), both always pick id 200;
    the sixth duplicate triggers the comparison, the lower-dos poi survives."""
    ops = []
    for call in range(1, 7):
        by = EI if call % 2 == 1 else POI
        ops += [suggest([1, 1, 1]), record(by, 10.0 if by == EI else 1.0)]
    out = trace(gt, MULTI, ops, active=[1, 1, 0])
    for call in range(1, 7):
        s = out[2 * (call - 1)]
        assert s.position == 1 and s.by == (EI if call % 2 == 1 else POI)
        if call < 6:
            assert s.duplicates[EI] == call and s.duplicates[POI] == call
            assert list(s.active) == [1, 1, 0]
    last = out[-1]
    assert list(last.active) == [0, 1, 0]  # ei skipped: dos(poi) < dos(ei)
    assert last.duplicates[POI] == 0       # counters consumed by the comparison


def test_multi_three_way_duplicates(gt):
    """All three functions agree: every suggestion conflicts with both others;
    with skip threshold 2 the third suggestion resolves the conflict to the
    lowest discounted observation score -- poi and (not yet recorded) lcb tie
    at 0, the earliest in fixed order wins (portfolio.hpp:222-236)."""
    ops, vals = [], {EI: 5.0, POI: 0.0, LCB: 1.0}
    for by in [EI, POI, LCB]:
        ops += [suggest([3, 3, 3]), record(by, vals[by])]
    out = trace(gt, MULTI, ops, skip=2)
    assert [out[i].duplicates[EI] for i in (0, 2)] == [1, 2]
    # third suggest: ei 3, poi 3, lcb 3 > 2 -> keep min dos among {ei, poi, lcb}:
    # dos(poi) == dos(lcb) == 0.0 < dos(ei) == 5.0 -> poi (earliest of the tie)
    assert list(out[4].active) == [0, 1, 0]
    assert list(out[4].duplicates) == [0, 0, 0]
    # with poi recording 1.0 instead, the unrecorded lcb (dos 0) is kept
    ops[3] = record(POI, 1.0)
    assert list(trace(gt, MULTI, ops, skip=2)[4].active) == [0, 0, 1]


def test_advanced_skip_then_promote_with_constant_scores(gt):
    """test_portfolio.cpp:166-207: constant observations (7, 10, 13); lcb is
    skipped in cycle 5 (resetting the others' counters), ei promoted in
    cycle 10."""
    value_of = {EI: 7.0, POI: 10.0, LCB: 13.0}
    ops, where = [], []
    for cycle in range(1, 11):
        for a in (EI, POI, LCB):
            if a == LCB and cycle > 5:
                continue
            if a == POI and cycle == 10:
                continue  # ei's record in cycle 10 promoted it
            ops.append(record(a, value_of[a]))
            where.append((cycle, a))
    out = trace(gt, ADVANCED, ops)
    changes = [(where[i], list(out[i].active)) for i in range(len(out))
               if list(out[i].active) != (list(out[i - 1].active) if i else [1, 1, 1])]
    assert changes == [((5, LCB), [1, 1, 0]), ((10, EI), [1, 0, 0])]
    hist = {a: [] for a in (EI, POI, LCB)}
    for i, (cycle, a) in enumerate(where):
        hist[a].append(value_of[a])
        assert out[i].dos[a] == dos_of(hist[a], 0.75)  # bit-exact: same IEEE operations


def test_advanced_promotion_after_qualifying_rounds(gt):
    """test_portfolio.cpp:208-239: eight cycles of identical scores change
    nothing; then poi lands below the band and is promoted on its fifth
    qualifying round."""
    ops = []
    for _ in range(8):
        ops += [record(EI, 10.0), record(POI, 10.0), record(LCB, 10.0)]
    warm = len(ops)
    for cycle in range(1, 6):
        ops += [record(EI, 10.0), record(POI, 2.0 if cycle == 1 else 8.0)]
        if cycle < 5:
            ops.append(record(LCB, 10.0))
    out = trace(gt, ADVANCED, ops)
    assert all(list(o.active) == [1, 1, 1] for o in out[:-1])
    assert list(out[-1].active) == [0, 1, 0]
    assert all(list(o.active) == [1, 1, 1] for o in out[:warm])


def test_trace_rejects_bad_config(gt):
    cfg = _lib.gtc_portfolio_config(MULTI, 0, 0.65, 0.1)
    out = (_lib.gtc_portfolio_state * 1)()
    ops = (_lib.gtc_portfolio_op * 1)()
    assert gt.load().gtc_portfolio_trace(0, C.byref(cfg), None, 1, ops, out) == _lib.GTC_ERR_CONFIG
