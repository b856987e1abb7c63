"""CPU-only checks: the synthetic input generator against the reference's,
the GEMM search space, and that the C-ABI library exports every symbol the
public header declares (no compute calls: there is no GPU here)."""
import ctypes as C
import pathlib
import re
import subprocess

import numpy as np
import pytest

from paper_2111_14991_b200 import synthetic

ROOT = pathlib.Path(__file__).resolve().parents[1]


def test_random_rough_bit_exact(golden):
    g = np.load(golden / "space_c3.npz")
    coords, ids, values = synthetic.random_rough([10, 10, 10, 10, 5, 2], 20261017, 0.3)
    np.testing.assert_array_equal(ids, g["ids"])
    np.testing.assert_array_equal(np.isnan(values), np.isnan(g["values"]))
    np.testing.assert_array_equal(values[~np.isnan(values)], g["values"][~np.isnan(g["values"])])
    assert int(np.isnan(values).sum()) == int(g["meta"][2])
    assert np.nanmin(values) == g["meta"][3]


def test_trajectory_spaces_bit_exact(golden):
    for f in sorted(golden.glob("traj_*.npz")):
        t = np.load(f)
        fn, grid = str(t["spec"][0]), [int(k) for k in str(t["spec"][1]).split("x")]
        seed, inv = int(t["spec"][2]), str(t["spec"][3])
        if fn == "random-rough":
            coords, ids, values = synthetic.random_rough(grid, seed, float(inv) if inv != "-" else 0.1)
        else:
            coords, ids, values = synthetic.rosenbrock_disc(grid, seed)
        np.testing.assert_array_equal(coords, t["coords"])
        np.testing.assert_array_equal(ids, t["ids"])
        np.testing.assert_array_equal(np.nan_to_num(values, nan=-1.0), np.nan_to_num(t["values"], nan=-1.0))


def test_gemm_space_matches_reference_enumeration(golden):
    """C1 GEMM space: 17,956 of 82,944 — canonical indices
    bit-exact against the reference restriction parser + enumeration."""
    g = np.load(golden / "space_gemm.npz")
    assert int(g["meta"][0]) == 17956 and int(g["meta"][2]) == 82944
    vals = [[16, 32, 64, 128], [16, 32, 64, 128], [32], [8, 16, 32], [8, 16, 32], [8, 16, 32],
            [8, 16, 32], [2], [1, 2, 4, 8], [1, 2, 4, 8], [0], [0], [0, 1], [0, 1], [32]]
    ranks = synthetic.grid_ranks([len(v) for v in vals])
    x = [np.asarray(v, dtype=np.float64)[ranks[:, j]] for j, v in enumerate(vals)]
    MWG, NWG, KWG, MDIMC, NDIMC, MDIMA, NDIMB, KWI, VWM, VWN = x[:10]
    ok = (np.fmod(KWG, KWI) == 0) & (np.fmod(MWG, MDIMC * VWM) == 0) & (np.fmod(NWG, NDIMC * VWN) == 0) \
        & (np.fmod(MWG, MDIMA * VWM) == 0) & (np.fmod(NWG, NDIMB * VWN) == 0) \
        & (np.fmod(KWG, (MDIMC * NDIMC) / MDIMA) == 0) & (np.fmod(KWG, (MDIMC * NDIMC) / NDIMB) == 0)
    idx = np.nonzero(ok)[0]
    np.testing.assert_array_equal(idx.astype(np.uint64), g["ids"])
    coords = synthetic.grid_coords([len(v) for v in vals], ranks[idx])
    np.testing.assert_array_equal(coords, g["coords"])


def _declared_symbols():
    text = (ROOT / "include" / "gridtune_cuda.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gtc_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(gt):
    lib = C.CDLL(str(gt.LIB_PATH))
    syms = _declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding covers exactly the declared surface
    from paper_2111_14991_b200 import _lib
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == syms


def test_library_is_sm100a(gt):
    out = subprocess.run(["cuobjdump", "--list-elf", str(gt.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_device(gt):
    """Without a GPU the compute entry points fail loudly (DeviceError)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(gt.DeviceError):
        gt.Space(np.zeros((10, 2)))
