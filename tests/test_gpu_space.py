"""Device search-space enumeration (gtc_space_enumerate, enum_kernels.cu)
against the UNMODIFIED reference's SearchSpace / EnumeratedSpace
(search_space.hpp:120-166,216-245; fixtures written by oracle/_ref/ref_tool):
canonical ids and normalised coordinates bit for bit, every well-formed
restriction of restrictions.json evaluated on the whole grid, the C1 GEMM
space, the empty-space error, and the resident space feeding a run."""
import json
import pathlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = pathlib.Path(__file__).parent / "golden"


def defs(gt, spec):
    return [gt.ParameterDef(p["name"], p["values"], gt.ParamKind[p["kind"]]) for p in spec]


@pytest.mark.parametrize("name", ["conv", "pnpoly", "typed", "ieee"])
def test_enumeration_matches_reference(gt, name):
    z = np.load(GOLDEN / f"enum_{name}.npz")
    spec = json.loads(str(z["spec"]))
    es = gt.SearchSpace(defs(gt, spec["params"]), spec["restrictions"]).enumerate()
    np.testing.assert_array_equal(es.ids, z["ids"])
    assert es.coords.tobytes() == np.ascontiguousarray(z["coords"]).tobytes()
    assert es.cartesian_size() == int(z["cartesian"][0])


def test_every_restriction_on_the_grid(gt):
    """Each well-formed restriction alone: the kept canonical indices are the
    reference's true bits (restriction.hpp:416-504 semantics incl. NaN/inf,
    fmod, string order, booleans)."""
    data = json.loads((GOLDEN / "restrictions.json").read_text())
    params = defs(gt, data["params"])
    checked = 0
    for case in data["cases"]:
        if not case["ok"]:
            continue
        want = np.nonzero(np.frombuffer(case["bits"].encode(), dtype=np.uint8) == ord("1"))[0]
        sp = gt.SearchSpace(params, [case["text"]])
        if len(want) == 0:
            with pytest.raises(gt.EmptySearchSpaceError):
                sp.enumerate()
        else:
            np.testing.assert_array_equal(sp.enumerate().ids, want.astype(np.uint64), err_msg=case["text"])
        checked += 1
    assert checked > 250


def test_gemm_space(gt):  # C1, PAPER.md:319-333 + Kernel Tuner restrictions
    z = np.load(GOLDEN / "space_gemm.npz")
    P = gt.ParameterDef
    params = [P("MWG", [16, 32, 64, 128]), P("NWG", [16, 32, 64, 128]), P("KWG", [32]),
              P("MDIMC", [8, 16, 32]), P("NDIMC", [8, 16, 32]), P("MDIMA", [8, 16, 32]), P("NDIMB", [8, 16, 32]),
              P("KWI", [2]), P("VWM", [1, 2, 4, 8]), P("VWN", [1, 2, 4, 8]), P("STRM", [0]), P("STRN", [0]),
              P("SA", [0, 1]), P("SB", [0, 1]), P("PRECISION", [32])]
    rs = ["KWG % KWI == 0", "MWG % (MDIMC * VWM) == 0", "NWG % (NDIMC * VWN) == 0", "MWG % (MDIMA * VWM) == 0",
          "NWG % (NDIMB * VWN) == 0", "KWG % ((MDIMC * NDIMC) / MDIMA) == 0", "KWG % ((MDIMC * NDIMC) / NDIMB) == 0"]
    es = gt.SearchSpace(params, rs).enumerate()
    assert es.n == 17956 and es.cartesian_size() == 82944
    np.testing.assert_array_equal(es.ids, z["ids"])
    assert es.coords.tobytes() == np.ascontiguousarray(z["coords"]).tobytes()


def test_empty_space(gt):
    case = json.loads((GOLDEN / "enum_errors.json").read_text())["empty"]
    with pytest.raises(gt.EmptySearchSpaceError, match=case["result"]["message"]):
        gt.SearchSpace(defs(gt, case["spec"]["params"]), case["spec"]["restrictions"]).enumerate()


def test_large_grid_and_run_on_enumerated_space(gt):
    """A 12.5M-point grid with restrictions, checked against a numpy restatement
    of the same IEEE arithmetic; then a GP run on the resident enumerated
    space predicts exactly like one on a space built from the same coordinates."""
    P = gt.ParameterDef
    vals = [list(range(1, 26)), [0.5 * i for i in range(20)], list(range(10)), [1, 2, 4, 8, 16],
            list(range(50)), [3, 5]]
    names = ["a", "b", "c", "d", "e", "f"]
    rs = ["a * b % 7 != 3", "(c + e) / d < 9.5 or f == 5", "not (a % 4 == 0 and e > 40)"]
    es = gt.SearchSpace([P(n, v) for n, v in zip(names, vals)], rs).enumerate()
    grids = np.meshgrid(*[np.array(v, dtype=np.float64) for v in vals], indexing="ij")
    a, b, c, d, e, f = [g.ravel() for g in grids]
    with np.errstate(all="ignore"):
        keep = (np.fmod(a * b, 7) != 3) & (((c + e) / d < 9.5) | (f == 5)) & ~((np.fmod(a, 4) == 0) & (e > 40))
    np.testing.assert_array_equal(es.ids, np.nonzero(keep)[0].astype(np.uint64))
    assert es.cartesian_size() == keep.size
    # the resident enumerated space drives a run exactly like explicit coordinates
    sub = np.arange(0, es.n, max(1, es.n // 40000))
    plain = gt.Space(es.coords[sub])
    kern = gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0)
    rng = np.random.default_rng(1)
    pos = rng.choice(len(sub), 30, replace=False)
    y = rng.random(30)
    r1 = gt.SurrogateRun(plain, kern, n_max=32)
    r1.fit(pos, y)
    m1, v1 = r1.predictions()
    r2 = gt.SurrogateRun(es, kern, n_max=32)
    r2.fit(sub[pos], y)
    m2, v2 = r2.predictions()
    assert m1.tobytes() == m2[sub].tobytes() and v1.tobytes() == v2[sub].tobytes()
