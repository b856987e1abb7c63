"""Initial-sample snap on the device (gtc_space_nearest) against a restatement
of draw_initial_sample's scan (sampling.hpp:98-117): squared distance summed
in parameter order without contraction, strict `<` (lowest position on ties);
compact (enumerated / few distinct values) and plain coordinate paths."""
import numpy as np
import pytest

from paper_2111_14991_b200 import synthetic

pytestmark = pytest.mark.gpu


def scan_nearest(coords, pts):
    out = []
    for p in pts:
        d2 = np.zeros(len(coords))
        for j in range(coords.shape[1]):  # sequential in j, like `d2 += diff * diff`
            diff = p[j] - coords[:, j]
            d2 = d2 + diff * diff
        out.append(int(np.argmin(d2)))  # first minimum = strict < scan
    return np.array(out)


def test_snap_on_grid_space_with_ties(gt):
    coords, ids, values = synthetic.random_rough([7, 5, 9, 4], 3, 0.0)
    space = gt.Space(coords)
    rng = np.random.default_rng(0)
    pts = rng.random((37, 4))
    # exact midpoints between neighbouring grid values: ties broken to the lower position
    pts[:5, 0] = 0.5 / 6 + np.arange(5) / 6
    pts[5:8] = coords[[3, 100, 500]]
    np.testing.assert_array_equal(space.nearest(pts), scan_nearest(coords, pts))


def test_snap_on_plain_coordinates(gt):
    rng = np.random.default_rng(1)
    coords = rng.random((70_001, 3))  # > 256 distinct values: the pass reads raw coordinates
    space = gt.Space(coords)
    pts = np.vstack([rng.random((20, 3)), coords[[0, 17, 70_000]]])
    np.testing.assert_array_equal(space.nearest(pts), scan_nearest(coords, pts))


def test_snap_on_enumerated_space(gt):
    P = gt.ParameterDef
    es = gt.SearchSpace([P("a", list(range(12))), P("b", [1, 2, 4, 8, 16, 32]), P("c", [0.5, 1.5, 2.5])],
                        ["a * b % 3 != 1"]).enumerate()
    rng = np.random.default_rng(2)
    pts = rng.random((50, 3))
    np.testing.assert_array_equal(es.nearest(pts), scan_nearest(es.coords, pts))
